cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for f in 80 96; do
LFM_TC_SMS_F=$f timeout 900 python bench.py --config c4 --steps 8 --warmup 2 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2r_c4_f$f.json 2> gpurun_out/r2r_c4_f$f.err; echo "c4 f$f rc=$?"
done
for b in 80 112; do
LFM_TC_SMS_F=80 LFM_TC_SMS_B=$b timeout 900 python bench.py --config c4 --steps 8 --warmup 2 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2r_c4_b$b.json 2> gpurun_out/r2r_c4_b$b.err; echo "c4 b$b rc=$?"
done
