"""Golden run of the reduced cfg4 multilevel solve (synth.make_cfg4_small)
with the REFERENCE evaluator (oracle/_ref/cfg4_solve_ref: the reference's
evaluate.cpp/lbfgs.cpp/solve.cpp compiled from /root/reference, 8 workers).
Writes cfg4_small_ref.json (stage reports) and cfg4_small_ref_psi.f64 (final
gauge-fixed potential).  Run in the build container."""
import os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "cfg4_prepare.py"), "/tmp/cfg4s", "small"], check=True)
env = dict(os.environ, RSOT_WORKERS="8", RSOT_DUMP_PSI=os.path.join(HERE, "cfg4_small_ref_psi.f64"))
out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "cfg4_solve_ref"), "/tmp/cfg4s", "1e-8", "1000"],
                     env=env, check=True, capture_output=True, text=True).stdout
open(os.path.join(HERE, "cfg4_small_ref.json"), "w").write(out)
print(out)
