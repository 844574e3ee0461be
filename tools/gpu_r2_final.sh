# end-of-session regression + sweep + ncu evidence; everything under gpurun_out/final_r2b/
O=${O:-gpurun_out/final_r2b}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -15 > $O/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
run() { name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?" >> $O/rc.log; }
run c5 --config c5
run c5_device --no-cpu-baseline --config c5 --weight-tier device
run c6 --no-cpu-baseline --config c6
run c6_device --no-cpu-baseline --config c6 --weight-tier device
run c2 --no-cpu-baseline --config c2
run c3 --no-cpu-baseline --config c3
run c3_kv4 --no-cpu-baseline --config c3 --kv-fmt int4
run c7 --no-cpu-baseline --config c7
run c1 --no-cpu-baseline --config c1
timeout 600 python bench.py --impl reference > $O/ref_c5.json 2> $O/ref_c5.err; echo "ref rc=$?" >> $O/rc.log
# ncu launch list of the default bench command past the weight generation (cold-cache, serialised: shares, not absolutes)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 1500 --csv --log-file $O/ncu_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cupti --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu-launch rc=$?" >> $O/rc.log
# full captures: the c5 decode GEMM (FC1, in-kernel fixup) and the c5 decode attention
bash tools/ncu_tm.sh > $O/ncu_tm.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 3 -c 1 -o $O/ncu_attn_c5 python tools/abench.py c5 > $O/ncu_attn.log 2>&1; echo "ncu-attn rc=$?" >> $O/rc.log
mv gpurun_out/ncu_tm_fc1.ncu-rep gpurun_out/ncu_tm_fc2.ncu-rep $O/ 2>/dev/null
cat $O/rc.log; tail -3 $O/gpu_suite.log; tail -1 $O/smoke.log
