cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -rs -x -k "frames_plan" 2>&1 | tail -3
for F in 16 32; do
timeout 900 python bench.py --config c5 --frames $F --steps 5 --warmup 2 > gpurun_out/r2n_c5_F$F.json 2>&1; echo "c5 F$F rc=$?"
done
LFM_MF_CHAIN=48 timeout 900 python bench.py --config c5 --frames 32 --steps 5 --warmup 2 > gpurun_out/r2n_c5_F32_ch48.json 2>&1; echo "c5 ch48 rc=$?"
