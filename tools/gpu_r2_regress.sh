# regression at HEAD: full GPU suite, smoke, default bench; logs under gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -25 > gpurun_out/regress_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/regress_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/regress_bench.json 2> gpurun_out/regress_bench.err
tail -3 gpurun_out/regress_suite.log gpurun_out/regress_smoke.log
head -c 600 gpurun_out/regress_bench.json
