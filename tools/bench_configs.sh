# bench lines for a list of configs (tool): CONFIGS="a b c" [ENVS] bash tools/bench_configs.sh
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{c}.json"))
except Exception as e:
    print(c, "FAILED", e); sys.exit()
r = d["roofline"]
print(f"{c}: {d['ms_per_step']:.3f} ms  {d['value']/1e6:.2f} M tok/s  dom {r['kernel']} {r['achieved']:.0f}/{r['peak']:.0f} {r['unit']} frac {r['frac']:.2f}  "
      f"dense {d.get('dense_context', {}).get('ms_per_step', float('nan')):.3f} ms  clocks {d['clocks']['sm_mhz']}")
PY
done
