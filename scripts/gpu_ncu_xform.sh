# ncu --set full of the tile-window transforms (register kernels) at c3, one iteration's worth of launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_step.py --iters 3 > gpurun_out/ncux_ps.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tile_reg_kernel" -s 24 -c 16 -o gpurun_out/ncu_xform python scripts/prof_step.py --iters 3 > gpurun_out/ncux_ncu.log 2>&1
echo "ncu rc=$?"
