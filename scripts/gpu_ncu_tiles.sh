cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_step.py --iters 2 > gpurun_out/ncu_ps.log 2>&1 && \
LFM_SERIAL=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"mac_f16_kernel|tcdir_kernel|r2c_tile_reg_kernel<27|c2r_tile_reg_kernel<27, 3" -s 10 -c 8 -o gpurun_out/ncu_full python scripts/prof_step.py --iters 2 > gpurun_out/ncu_ncu_full.log 2>&1
echo "full rc=$?"
