cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for i in 1 2 3; do
for m in 0 1; do
  if [ $m = 1 ]; then export LFM_STAGE_PREFORK=1; else unset LFM_STAGE_PREFORK; fi
  timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2j_$m.$i.json 2>/dev/null; echo "pre=$m rc=$?"
done; done
