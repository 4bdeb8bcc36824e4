cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
python scripts/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dir_" -s 3 -c 3 -o gpurun_out/prof_dir python scripts/prof_step.py --iters 2 > gpurun_out/ncu_dir.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_dir.log; cat gpurun_out/prof_plain.log
