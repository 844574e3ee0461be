# default bench line (c5) + device-tier c5/c6 lines under gpurun_out/bench_r2b/
mkdir -p gpurun_out/bench_r2b
timeout 900 python bench.py > gpurun_out/bench_r2b/c5.json 2> gpurun_out/bench_r2b/c5.err; echo c5 rc=$?
timeout 900 python bench.py --no-cpu-baseline --config c5 --weight-tier device > gpurun_out/bench_r2b/c5_device.json 2> gpurun_out/bench_r2b/c5_device.err; echo c5d rc=$?
timeout 900 python bench.py --no-cpu-baseline --config c6 --weight-tier device > gpurun_out/bench_r2b/c6_device.json 2> gpurun_out/bench_r2b/c6_device.err; echo c6d rc=$?
