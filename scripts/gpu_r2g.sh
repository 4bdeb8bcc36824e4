cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_c3_parity.py -q -m gpu -rs -k c3g13 2>&1 | tail -3
for cfg in "8 2" "8 4" "16 4"; do set -- $cfg
  LFM_MT_PREP=$1 LFM_MT_PG=$2 timeout 600 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 > gpurun_out/r2g_c5_$1_$2.json 2>&1; echo "c5 $1 $2 rc=$?"
done
LFM_MT_PREP=16 LFM_MT_PG=4 timeout 600 python bench.py --config c5 --frames 8 --steps 5 --warmup 2 > gpurun_out/r2g_c5_F8.json 2>&1; echo "c5 F8 rc=$?"
LFM_MT_PREP=16 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rs -k batched 2>&1 | tail -3
