cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
CMD="python bench.py --config c5 --frames 16 --steps 1 --warmup 1"
$CMD > gpurun_out/c5_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fmb_tc|bwd_mac_batch" -c 2 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_c5.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_c5.log
