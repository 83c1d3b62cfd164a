# Shared main-solve inputs for the C3 / C4 full parity (eps' warm potentials + basis, made
# on the GPU), then the GPU's own main solves in both accept modes (tools/full_parity.py).
set -x
for cfg in C3 C4; do
  tag=$(echo $cfg | tr 'A-Z' 'a-z')
  SKNR_PARITY_CFG=$cfg timeout 900 python tools/c4_full_parity.py gpu > gpurun_out/${tag}_inputs.log 2>&1; echo inputs_$cfg=$?
  mkdir -p ${tag}_full_inputs && cp gpurun_out/${tag}_full/inputs.npz ${tag}_full_inputs/
  SKNR_PARITY_CFG=$cfg timeout 900 python tools/full_parity.py gpu > gpurun_out/${tag}_gpu.log 2>&1; echo gpu_$cfg=$?
done
