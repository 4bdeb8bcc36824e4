# TC-path check: focused GPU tests, then quick c3 bench variants
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-tc or projections or c2_operators or adjoint}" 2>&1 | tail -5
bash scripts/gpu_bench_quick.sh "$@"
