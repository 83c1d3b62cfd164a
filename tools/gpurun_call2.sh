set -x
timeout 600 python tools/diag_stable_c3.py C3 > gpurun_out/diag_c3.log 2>&1; echo diag=$?
bash tools/gpurun_parity_inputs.sh
