set -x
timeout 900 python tools/variant_check.py 5 40 46 50 52 53 54 59 60 61 62 63 64 > gpurun_out/variant_check4.log 2>&1; echo vc=$?
timeout 600 python tools/tune_lse.py 4 5 40 46 50 51 52 53 54 55 56 57 58 59 60 61 62 63 64 > gpurun_out/tune4.log 2>&1; echo tune=$?
timeout 1500 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > gpurun_out/gputest4.log 2>&1; echo pytest=$?
