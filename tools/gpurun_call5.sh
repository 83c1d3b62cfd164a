set -x
timeout 900 python tools/variant_check.py 4 62 65 66 67 68 69 > gpurun_out/variant_check5.log 2>&1; echo vc=$?
timeout 600 python tools/tune_lse.py 4 5 46 62 65 66 67 68 69 > gpurun_out/tune5.log 2>&1; echo tune=$?
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/gputest5.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke5.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench=$?
timeout 300 python tools/profile_lse.py 2 > gpurun_out/p2.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:pts_sum12_kernel' -s 2 -c 1 -o gpurun_out/ncu_lse_sum12_r02 python tools/profile_lse.py 2 > gpurun_out/ncu_lse_sum12_r02.log 2>&1; echo ncu=$?
