# usage: bash scripts/gpu_ncu_k.sh <kernel-regex> <skip> <count> [prof_step args]
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
K=$1; S=$2; C=$3; shift 3
python scripts/prof_step.py --iters 2 "$@" > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $C -o gpurun_out/prof_k python scripts/prof_step.py --iters 2 "$@" > gpurun_out/ncu_k.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_k.log
