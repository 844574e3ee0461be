# full GPU suite file by file (each under its own timeout), smoke, default bench; logs in gpurun_out/
rm -f gpurun_out/suite_safe.log
for f in tests/test_gpu_*.py; do
  timeout 900 python -m pytest $f -q -m gpu -x 2>&1 | tail -2 | sed "s|^|$f: |" >> gpurun_out/suite_safe.log
done
cat gpurun_out/suite_safe.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_safe.json 2> gpurun_out/bench_safe.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_safe.json')); print(d['value'], d['e2e']['value'], d['setup']['prefill_s'], d['prefill_kernels'], d['roofline']['frac'], d['clocks'])"
