cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_step.py --iters 2 --flags 4096 > gpurun_out/t5_ps.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"mac_f16_kernel|r2c_tile_reg_kernel|c2r_tile_reg_kernel" -s 6 -c 5 -o gpurun_out/t5_full python scripts/prof_step.py --iters 2 --flags 4096 > gpurun_out/t5_ncu_full.log 2>&1
echo "full rc=$?"
