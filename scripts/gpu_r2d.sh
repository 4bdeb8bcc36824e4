cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rs -x -k "partitions or column_ranges or projections or auto_stop" 2>&1 | tail -4
for k in 0 3 5 7 10; do
  LFM_PLAN_MOVE=$k LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2d_move$k.json 2> gpurun_out/r2d_move$k.err; echo "move $k rc=$?"
done
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2d_auto.json 2> gpurun_out/r2d_auto.err; echo "auto rc=$?"
