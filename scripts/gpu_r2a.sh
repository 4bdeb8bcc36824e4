cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
nproc
timeout 2000 python -m pytest tests -q -m gpu -rs --durations=15 -k "not c3_auto and not c3g13 and not multigpu" 2>&1 | tail -30
for i in 1 2; do LFM_MT_PG=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k batched 2>&1 | tail -2; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 > gpurun_out/r2a_c5_pg2.json 2>&1; echo "c5 rc=$?"
LFM_MT_PG=4 timeout 600 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 > gpurun_out/r2a_c5_pg4.json 2>&1; echo "c5 pg4 rc=$?"
