#!/bin/bash
# GPU-box host run of the C3 oracle's own main-solve trajectories (both accept modes in
# parallel, 8 threads each); checkpoints land in gpurun_out/c3_r02 and travel back.
# A gpurun call is capped at an hour: the oracles stop themselves after SECS seconds and
# the next call resumes from the checkpoints copied into c3_full_inputs/box/ (gpurun_out/
# does not travel to the box).
# usage: cp gpurun_out/c3_r02/oracle_*.npz c3_full_inputs/box/ ; gpurun --timeout 3600 -- bash tools/gpurun_c3_oracle.sh
SECS=${SECS:-3300}
export SKNR_PARITY_CFG=C3 SKNR_PARITY_STATE=gpurun_out/c3_r02 SKNR_PARITY_CHUNK=20 ORACLE_THREADS=8
mkdir -p gpurun_out/c3_r02
nproc > gpurun_out/c3_r02/host.txt
cp c3_full_inputs/box/oracle_*.npz gpurun_out/c3_r02/ 2>/dev/null
for mode in stable literal; do
  timeout "$SECS" python tools/full_parity.py oracle $mode >> gpurun_out/c3_r02/oracle_$mode.log 2>&1 &
done
wait
tail -2 gpurun_out/c3_r02/oracle_*.log
