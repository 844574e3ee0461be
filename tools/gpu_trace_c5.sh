timeout 600 python tools/trace_step.py --config c5 --tier device --steps 2 --kprof 0 > gpurun_out/trace_c5_dev.json 2> gpurun_out/trace_c5_dev.err
timeout 300 python tools/abench.py c5 > gpurun_out/abench_c5.log 2>&1
