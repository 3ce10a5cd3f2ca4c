cd $GRAFT_REPO_ROOT 2>/dev/null || true
for v in old new; do echo "== $v"; RSOT_LIB_PATH=paper_2507_23602_b200/lib/var_$v.so timeout 600 python tools/trunc_timing.py cfg5 cfg3 2>&1 | tail -2; done
echo "== new, persist off"; RSOT_CUDA_L2_PERSIST=0 RSOT_LIB_PATH=paper_2507_23602_b200/lib/var_new.so timeout 600 python tools/trunc_timing.py cfg5 cfg3 2>&1 | tail -2
