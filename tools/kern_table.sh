# Per-kernel table of one config (tool): CONFIG=bert [ENV="A=1"] bash tools/kern_table.sh
env $ENV timeout 300 python bench.py --config ${CONFIG:-bert} --steps 20 --warmup 5 --no-cpu-baseline --no-e2e ${EXTRA} > gpurun_out/kt.json 2>/dev/null
python - "$ENV" <<'PY'
import json, sys
d = json.load(open("gpurun_out/kt.json"))
print(f"== {d['config'].get('workload')} [{sys.argv[1] or 'default'}] {d['ms_per_step']:.4f} ms/step  clk {d['clocks']['sm_mhz']}  dense {d.get('dense_context', {})}")
tot = 0
for n, v in d["kernels"].items():
    tot += v["ms_per_launch"] * v.get("launches_per_step", 1)
    print(f"  {n:24s} {v['ms_per_launch']*1e3:9.1f} us  x{v.get('launches_per_step', 1)}")
print(f"  sum of kernels {tot*1e3:.1f} us")
PY
