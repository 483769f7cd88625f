# GPU validation pass (tool): bench line + full -m gpu suite (+ optional reference arm); outputs under gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 400 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
if [ -n "$REF" ]; then timeout 400 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?; fi
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gputests.log
