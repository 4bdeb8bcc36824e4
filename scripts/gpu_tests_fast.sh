cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -m gpu -rs -k "$1" 2>&1 | tail -25
