# round-end evidence: full GPU tests, default bench (with cpu baseline), ncu launch list of the bench command,
# ncu --set full of the dominant kernels (fwd_mac, bwd_mac, tcdir_kernel)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_final.json').read().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
# launch list of 4 RL iterations (prof_step.py); the plan's first kernels on each green context are skipped
# (--launch-skip: ncu cannot prepare the very first kernel of a fresh green context), and the same one after the other
python scripts/prof_step.py --iters 4 > gpurun_out/ps_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 89 -c 200 --csv --log-file gpurun_out/launches.csv python scripts/prof_step.py --iters 4 > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?"
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 89 -c 200 --csv --log-file gpurun_out/launches_serial.csv python scripts/prof_step.py --iters 4 > gpurun_out/ncu_launch_serial.log 2>&1
echo "launch-list serial rc=$?"
python scripts/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"mac_kernel|tcdir_kernel" -s 6 -c 4 -o gpurun_out/prof_final python scripts/prof_step.py --iters 2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
