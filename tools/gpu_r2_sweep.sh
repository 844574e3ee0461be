# end-of-round sweep: every config's bench line (JSON under gpurun_out/sweep_r2/)
mkdir -p gpurun_out/sweep_r2
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/sweep_r2/$name.json 2> gpurun_out/sweep_r2/$name.err; echo "$name rc=$?"; }
run c5 --config c5
run c6 --config c6
run c7 --config c7
run c2 --config c2
run c3 --config c3
run c3_kv4 --config c3 --kv-fmt int4
run c6_device --config c6 --weight-tier device
run c5_device --config c5 --weight-tier device
run c1 --config c1
timeout 600 python bench.py --impl reference > gpurun_out/sweep_r2/ref_c5.json 2> gpurun_out/sweep_r2/ref_c5.err; echo ref rc=$?
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/sweep_r2/*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unparsable", e); continue
    s = d.get("setup", {})
    print(f.split("/")[-1], round(d.get("value", 0), 2), d.get("unit"), "ms/step", round(d.get("ms_per_step", 0), 2),
          "link", round((d.get("link_roofline") or {}).get("frac", 0) or 0, 3), "busy", round((d.get("busy") or {}).get("union", 0) or 0, 4),
          "ttft", s.get("prefill_s"), "pf", {k: round(v.get("tflops", 0), 1) for k, v in (d.get("prefill_kernels") or {}).items()})
PY
