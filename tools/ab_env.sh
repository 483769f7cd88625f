# A/B of environment knobs on one config (tool): ENVS="A=1 B=2;C=3" CONFIG=llama_scale bash tools/ab_env.sh
IFS=';' read -ra SETS <<< "$ENVS"
for e in "" "${SETS[@]}"; do
  env $e timeout 300 python bench.py --config ${CONFIG:-llama_scale} --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/ab.json 2>/dev/null
  python - "$e" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
k = d["kernels"]
print(f"[{sys.argv[1] or 'default'}] {d['ms_per_step']:.3f} ms  " + " ".join(f"{n.replace('tc_','')}={v['ms_per_launch']:.3f}" for n, v in k.items() if v['ms_per_launch'] > 0.05) + f"  clk {d['clocks']['sm_mhz']}")
PY
done
