#!/bin/bash
# GPU-box host run of the C3 oracle's own main-solve trajectories (both accept modes in
# parallel, 8 threads each); checkpoints land in gpurun_out/c3_r02 and travel back.
# usage: gpurun --timeout 9000 -- bash tools/gpurun_c3_oracle.sh
export SKNR_PARITY_CFG=C3 SKNR_PARITY_STATE=gpurun_out/c3_r02 SKNR_PARITY_CHUNK=20 ORACLE_THREADS=8
mkdir -p gpurun_out/c3_r02
nproc > gpurun_out/c3_r02/host.txt
python tools/full_parity.py oracle stable > gpurun_out/c3_r02/oracle_stable.log 2>&1 &
python tools/full_parity.py oracle literal > gpurun_out/c3_r02/oracle_literal.log 2>&1 &
wait
tail -2 gpurun_out/c3_r02/oracle_*.log
