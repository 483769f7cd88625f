# GPU validation pass (tool): bench line + full -m gpu suite; outputs under gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gputests.log
