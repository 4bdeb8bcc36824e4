# FFT-kernel change check: focused parity tests, c5 + c3 bench, ncu of the coarse transforms
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-projections or rl_tiny or c2_operators or batched or isra or fft or smoke}" 2>&1 | tail -4
FRAMES=16 bash scripts/gpu_c5.sh
bash scripts/gpu_bench_quick.sh
bash scripts/gpu_ncu_fft.sh
