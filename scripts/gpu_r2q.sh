cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
python scripts/prof_frames.py --config c3 --frames 8 --iters 1 > gpurun_out/r2q_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2q_launches_frames.csv python scripts/prof_frames.py --config c3 --frames 8 --iters 1 > gpurun_out/r2q_ncu.log 2>&1
echo "list rc=$?"
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2q_c4.json 2> gpurun_out/r2q_c4.err; echo "c4 rc=$?"
