# usage: bash tools/gpurun_c3_seg.sh K0 K1 [gpu]   (C3 main-solve parity segment, < 1 h)
export SKNR_PARITY_CFG=C3
mkdir -p gpurun_out/c3_full c3_full_inputs
if [ "$3" = "gpu" ]; then
  timeout 300 python tools/c4_full_parity.py gpu > gpurun_out/c3_full/gpu.log 2>&1
  cp gpurun_out/c3_full/inputs.npz c3_full_inputs/
fi
timeout 3000 python tools/c4_full_parity.py segment $1 $2 > gpurun_out/c3_full/seg_$1.log 2>&1
tail -3 gpurun_out/c3_full/seg_$1.log
