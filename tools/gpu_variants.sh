for v in ${VARIANTS}; do echo "== $v"; RSOT_LIB_PATH=$v timeout 300 python tools/trunc_timing.py ${CFGS:-cfg5}; done
