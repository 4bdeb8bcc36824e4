# ncu launch list of 2 c3 RL iterations (prof_step.py) with SM partitions, then one after the other (LFM_SERIAL=1)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
python scripts/prof_step.py --iters 2 > gpurun_out/ps_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_part.csv python scripts/prof_step.py --iters 2 > gpurun_out/ncu_launch_part.log 2>&1
echo "launch-list partitions rc=$?"; tail -3 gpurun_out/ncu_launch_part.log
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_serial.csv python scripts/prof_step.py --iters 2 > gpurun_out/ncu_launch_serial.log 2>&1
echo "launch-list serial rc=$?"; tail -3 gpurun_out/ncu_launch_serial.log
