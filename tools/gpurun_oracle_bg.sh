#!/bin/bash
# One gpurun call = GPU work in the foreground + the long oracle trajectories of
# tools/full_parity.py on the box's host cores in the background (a gpurun call is capped
# at an hour, so the oracles stop themselves after SECS seconds and resume next call from
# the checkpoints copied into {c3,c4}_full_inputs/box/ -- gpurun_out/ does not travel).
#
# usage: SECS=3300 JOBS="C3:stable:6 C3:literal:6" gpurun --timeout 3600 -- \
#            bash tools/gpurun_oracle_bg.sh 'python -m pytest tests -m gpu -q -x'
# before the next call:  cp gpurun_out/c3_r02/oracle_*.npz c3_full_inputs/box/
SECS=${SECS:-3300}
JOBS=${JOBS:-"C3:stable:8 C3:literal:8"}
start=$(date +%s)
for job in $JOBS; do
  IFS=: read -r cfg mode threads <<< "$job"
  tag=$(echo "$cfg" | tr 'A-Z' 'a-z')
  mkdir -p gpurun_out/${tag}_r02
  cp ${tag}_full_inputs/box/oracle_${mode}.npz gpurun_out/${tag}_r02/ 2>/dev/null
  nproc > gpurun_out/${tag}_r02/host.txt
  SKNR_PARITY_CFG=$cfg SKNR_PARITY_STATE=gpurun_out/${tag}_r02 SKNR_PARITY_CHUNK=${CHUNK:-10} ORACLE_THREADS=$threads \
    timeout "$SECS" python tools/full_parity.py oracle $mode >> gpurun_out/${tag}_r02/oracle_$mode.log 2>&1 &
done
for cmd in "$@"; do
  echo "=== $cmd"
  bash -c "$cmd"
  echo "=== rc=$? after $(( $(date +%s) - start )) s"
done
wait
for job in $JOBS; do
  IFS=: read -r cfg mode threads <<< "$job"
  tag=$(echo "$cfg" | tr 'A-Z' 'a-z')
  echo "--- $cfg $mode"; tail -1 gpurun_out/${tag}_r02/oracle_$mode.log
done
