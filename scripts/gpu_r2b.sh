cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 120 ./scripts/tc_f16_test 2>&1 | tail -14
timeout 2000 python -m pytest tests -q -m gpu -rs -x --durations=5 -k "not c3_auto and not c3g13 and not multigpu" 2>&1 | tail -30
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
LFM_MT_PG=2 timeout 600 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 > gpurun_out/r2b_c5_pg2.json 2>&1; echo "c5 rc=$?"
LFM_MT_PG=4 timeout 600 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 > gpurun_out/r2b_c5_pg4.json 2>&1; echo "c5 pg4 rc=$?"
