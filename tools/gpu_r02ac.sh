mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02ac_ref_reference.json 2>&1
mv baseline/_ref /tmp/_ref_hidden
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02ac_ref_port.json 2>&1
mv /tmp/_ref_hidden baseline/_ref
python - <<'PY'
import json
for k in ("reference", "port"):
    d = json.loads(open(f"gpurun_out/r02ac_ref_{k}.json").read().strip().splitlines()[-1])
    m, e = d["measured"], d["extrapolated"]
    print(k, d["cpu_baseline"]["kind"], "value", round(d["value"], 1), "s/sample", round(m["s_per_sample"], 3),
          "per-it", {a: round(b * 1e3, 3) for a, b in e["per_iteration_s_at_sample"].items()},
          "asm+corr", round(e["assembly_correction_s_at_sample"], 3), "setup", round(m["setup_s"], 1))
PY
