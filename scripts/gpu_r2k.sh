cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
FRAMES=16 timeout 300 python scripts/sanitize_batch.py > gpurun_out/r2k_plain.log 2>&1 && \
FRAMES=16 timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 50 python scripts/sanitize_batch.py > gpurun_out/r2k_racecheck.log 2>&1
echo "racecheck rc=$?"
tail -5 gpurun_out/r2k_racecheck.log
