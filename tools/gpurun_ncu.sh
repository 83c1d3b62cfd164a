# usage: bash tools/gpurun_ncu.sh <which> <kernel-regex> <skip> <outname>
which=$1; rx=$2; skip=$3; out=$4
timeout 300 python tools/profile_lse.py $which > gpurun_out/${out}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:$rx" -s $skip -c 1 -o gpurun_out/$out python tools/profile_lse.py $which > gpurun_out/${out}_ncu.log 2>&1
echo "ncu rc=$?"
tail -4 gpurun_out/${out}_ncu.log
