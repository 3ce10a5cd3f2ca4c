# GPU cfg4 stages from the same stage-entry potentials as the CPU reference
# runs, with one line per evaluation (trajectory comparison).
mkdir -p gpurun_out/c4t
python tools/cfg4_prepare.py /tmp/cfg4 > /dev/null
for st in "fine 1e-4 psi_fine_1e-04" "coarse 1e-2 psi_coarse_1e-02" "coarse 0.1 psi_coarse_1e-01" "fine 1e-3 psi_fine_1e-03"; do
  set -- $st
  RSOT_CUDA_EVAL_LOG=1 timeout 600 paper_2507_23602_b200/lib/cfg4_solve /tmp/cfg4 --stage $1 $2 build/c4psi/$3.f64 1e-8 1000 \
    > gpurun_out/c4t/${1}_$2.json 2> gpurun_out/c4t/${1}_$2.err; echo $1 $2 rc=$?
done
