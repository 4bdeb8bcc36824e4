cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?"
python scripts/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"mac_kernel|r2c_kernel|c2r_kernel|metric" -s 9 -c 8 -o gpurun_out/prof_c3 python scripts/prof_step.py --iters 2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -5 gpurun_out/ncu_full.log
