# focused GPU tests, quick c3 bench, ncu launch list of the bench command (-> gpurun_out/launches.csv)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-tc or projections or c2_operators or adjoint or rl_tiny or isra}" 2>&1 | tail -3
bash scripts/gpu_bench_quick.sh
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-calls 1"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?"
python scripts/launch_table.py gpurun_out/launches.csv
