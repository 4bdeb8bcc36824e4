# dev A/B of the tcgen05 ring depths (kASlots / kBSlots) in one call: rebuilds on the box between variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
F=paper_2208_11422_b200/csrc/kernels_tcdir.cu
run() {
  python -m paper_2208_11422_b200.build > /dev/null 2>&1
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); c=d['config']
print('$1', round(d['value'],2), d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"
}
cp $F /tmp/tcdir_orig.cu
for r in 1 2; do
  cp /tmp/tcdir_orig.cu $F; run "A2B5"
  sed -i 's/^constexpr int kASlots = 2;/constexpr int kASlots = 3;/; s/^constexpr int kBSlots = 5;/constexpr int kBSlots = 4;/' $F; run "A3B4"
done
cp /tmp/tcdir_orig.cu $F
