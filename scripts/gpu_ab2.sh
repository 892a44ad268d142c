cd $GRAFT_REPO_ROOT
LIBS="${ABLIBS}" CFGS="7:4 7:3" bash scripts/gpu_ab.sh 2>&1 | grep -v "^$"
CONFIG=cjm9_16384 COUNT=600 LIBS="${ABLIBS}" CFGS="7:4" bash scripts/gpu_ab.sh 2>&1 | grep -v "^$"
