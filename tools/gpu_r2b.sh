set -u
out=gpurun_out; mkdir -p $out
(timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_r2b.txt 2>&1; echo "exit $?" >> $out/pytest_r2b.txt)
tail -3 $out/pytest_r2b.txt
timeout 600 python tools/w1_compare.py 200 200 1000 2000 > $out/w1_r2b.jsonl 2> $out/w1_r2b.err; cat $out/w1_r2b.jsonl; tail -3 $out/w1_r2b.err
for s in mnist fmnist imdb; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_bits_kernel -s 3 -c 1 -o $out/prof_eval_${s}_r2b -f python tools/eval_bench.py $s > $out/ncu_eval_${s}_r2b.txt 2>&1
  tail -2 $out/ncu_eval_${s}_r2b.txt
done
