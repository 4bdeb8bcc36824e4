cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 3 --cpu-rows 48 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "rc=$?"
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
