# c5 bench (N=1), launcher test with 2 ranks on one GPU (c1), reference arm c5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.out 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
tail -c 600 gpurun_out/bench_c5.err
python bench.py --gpus 2 --allow-shared-gpu --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1_n2.out 2> gpurun_out/bench_c1_n2.err; echo "c1 n2 rc=$?"
tail -c 1500 gpurun_out/bench_c1_n2.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_c5.out 2> gpurun_out/bench_ref_c5.err; echo "ref rc=$?"
