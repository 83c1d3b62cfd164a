set -x
timeout 600 python tools/tune_lse.py 400 401 402 403 404 405 > gpurun_out/tune7.log 2>&1; echo tune=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stable or full_size or facade or sharded or householder or coupling or newton" > gpurun_out/gputest7.log 2>&1; echo pytest=$?
timeout 300 python tools/c2_anneal_parity.py > gpurun_out/c2_7.log 2>&1; echo c2=$?
timeout 900 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench=$?
