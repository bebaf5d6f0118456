mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "sequential or dropin or mirror or golden or w1 or determin or jump or regress or smoke or cli or driver" > gpurun_out/seq_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/seq_pytest.txt; tail -2 gpurun_out/seq_pytest.txt
timeout 600 python tools/seq_time.py mnist 500 > gpurun_out/seq_mnist.json 2>&1; cat gpurun_out/seq_mnist.json
timeout 600 python tools/seq_time.py imdb 100 > gpurun_out/seq_imdb.json 2>&1; cat gpurun_out/seq_imdb.json
timeout 600 python tools/w1_time.py > gpurun_out/w1_time.json 2>&1; cat gpurun_out/w1_time.json
