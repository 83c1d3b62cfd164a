# usage: bash tools/gpurun_c4_seg.sh K0 K1   (one C4 parity segment, < 1 h)
mkdir -p gpurun_out/c4_full
nproc
timeout 3300 python tools/c4_full_parity.py segment $1 $2 > gpurun_out/c4_full/seg_$1.log 2>&1
tail -4 gpurun_out/c4_full/seg_$1.log
