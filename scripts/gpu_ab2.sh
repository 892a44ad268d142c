cd $GRAFT_REPO_ROOT
LIBS="build/var/libcjm_base.so paper_1705_00103_b200/libcjm.so" CFGS="7:3" bash scripts/gpu_ab.sh 2>&1 | grep -v "^$"
CONFIG=cjm9_16384 COUNT=600 LIBS="build/var/libcjm_base.so paper_1705_00103_b200/libcjm.so" CFGS="7:4" bash scripts/gpu_ab.sh 2>&1 | grep -v "^$"
