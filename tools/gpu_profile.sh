# ncu evidence for one LLaMA-scale step (tool): launch list of the bench command + --set full of one step
# TAG names the outputs (default r02): gpurun_out/${TAG}_launches.csv, gpurun_out/${TAG}_step_full.ncu-rep
TAG=${TAG:-r02}
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/${TAG}_launches_bench.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"tc_|combine_kernel|bucket_|topk_hist|tile_sched|dwr_reduce" -s 15 -c 15 -o gpurun_out/${TAG}_step_full \
    python bench.py --steps 1 --warmup 1 --no-graph --no-profile --no-e2e --no-cpu-baseline --no-dense > gpurun_out/${TAG}_step_full.log 2>&1; echo full rc=$?
