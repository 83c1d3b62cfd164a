#!/bin/bash
# Full-size oracle-own main-solve parity (tools/full_parity.py), one gpurun call:
#   1. (first call only) the shared inputs -- eps' warm potentials and top_modes basis --
#      and the GPU's own trajectories in both accept modes, for every config in CFGS
#      whose {c3,c4}_full_inputs/inputs.npz is missing; copied to gpurun_out/ to travel back;
#   2. the oracle's own trajectory (JOBS = "CFG:mode:threads ...") on the box's host cores
#      in the background for SECS seconds, resumed from {cfg}_full_inputs/oracle_<mode>.npz;
#   3. the commands given as arguments, in the foreground (GPU work) -- with ORACLE_AFTER=1
#      BEFORE the oracles start, so that timings and CPU baselines see an idle host.
#      A job may carry a niceness as a 4th field ("C4:literal:16:19": runs on what the
#      other jobs leave idle).
# Before the next call:  cp gpurun_out/c4_r02/oracle_*.npz c4_full_inputs/
SECS=${SECS:-3300}
CFGS=${CFGS:-"C4 C3"}
JOBS=${JOBS:-"C4:stable:16"}
start=$(date +%s)
nproc > gpurun_out/host_nproc.txt
for cfg in $CFGS; do
  tag=$(echo "$cfg" | tr 'A-Z' 'a-z')
  mkdir -p gpurun_out/${tag}_r02 ${tag}_full_inputs
  if [ ! -f ${tag}_full_inputs/inputs.npz ]; then
    SKNR_PARITY_CFG=$cfg timeout 600 python tools/c4_full_parity.py gpu > gpurun_out/${tag}_r02/inputs.log 2>&1
    cp gpurun_out/${tag}_full/inputs.npz ${tag}_full_inputs/inputs.npz
    SKNR_PARITY_CFG=$cfg timeout 600 python tools/full_parity.py gpu > gpurun_out/${tag}_r02/gpu.log 2>&1
    echo "inputs $cfg rc=$? after $(( $(date +%s) - start )) s"
  fi
done
run_cmds() {
  for cmd in "$@"; do
    echo "=== $cmd"
    bash -c "$cmd"
    echo "=== rc=$? after $(( $(date +%s) - start )) s"
  done
}
if [ "${ORACLE_AFTER:-0}" = "1" ]; then run_cmds "$@"; fi
for job in $JOBS; do
  IFS=: read -r cfg mode threads prio <<< "$job"
  tag=$(echo "$cfg" | tr 'A-Z' 'a-z')
  mkdir -p gpurun_out/${tag}_r02
  cp ${tag}_full_inputs/oracle_${mode}.npz gpurun_out/${tag}_r02/ 2>/dev/null
  SKNR_PARITY_CFG=$cfg SKNR_PARITY_STATE=gpurun_out/${tag}_r02 SKNR_PARITY_CHUNK=${CHUNK:-1} ORACLE_THREADS=$threads \
    nice -n ${prio:-0} timeout "$SECS" python tools/full_parity.py oracle $mode >> gpurun_out/${tag}_r02/oracle_$mode.log 2>&1 &
done
if [ "${ORACLE_AFTER:-0}" != "1" ]; then run_cmds "$@"; fi
wait
for job in $JOBS; do
  IFS=: read -r cfg mode threads prio <<< "$job"
  tag=$(echo "$cfg" | tr 'A-Z' 'a-z')
  echo "--- $cfg $mode"; tail -2 gpurun_out/${tag}_r02/oracle_$mode.log
done
