# regression after the plain-launch attention change: full GPU suite + smoke + c5/c6 lines (both tiers) + c2/c3
O=gpurun_out/final_r2c; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -6 > $O/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
run() { name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?" >> $O/rc.log; }
run c5 --config c5
run c5_device --no-cpu-baseline --config c5 --weight-tier device
run c6 --no-cpu-baseline --config c6
run c6_device --no-cpu-baseline --config c6 --weight-tier device
run c2 --no-cpu-baseline --config c2
run c3 --no-cpu-baseline --config c3
run c3_kv4 --no-cpu-baseline --config c3 --kv-fmt int4
cat $O/rc.log; tail -2 $O/gpu_suite.log; tail -1 $O/smoke.log
