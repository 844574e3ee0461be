# final check at HEAD: full GPU suite, smoke, default bench line
O=${O:-gpurun_out/final_check}; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -4 > $O/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/c5.json 2> $O/c5.err; echo "bench rc=$?"
tail -2 $O/gpu_suite.log; tail -1 $O/smoke.log
