cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 300 python tools/graph_vs_eager.py --config c2_b8 --mode prefill --steps 30; done
for i in 1 2; do bash tools/exp.sh c2_b8 2::8; done
