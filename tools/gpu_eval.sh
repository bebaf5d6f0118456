# Inference check + timing + one ncu capture per shape: bash tools/gpu_eval.sh <tag>
set -u
tag=$1; out=gpurun_out; mkdir -p $out
(timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "inference or refresh or parity or edge or regress or dropin or predict or sums" > $out/pytest_$tag.txt 2>&1; echo "exit $?" >> $out/pytest_$tag.txt)
tail -3 $out/pytest_$tag.txt
timeout 600 python tools/eval_bench.py > $out/eval_$tag.jsonl 2> $out/eval_$tag.err; cat $out/eval_$tag.jsonl; tail -3 $out/eval_$tag.err
if [ "${NCU:-1}" = "1" ]; then
for s in mnist fmnist imdb; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_bits_kernel -s 3 -c 1 -o $out/prof_eval_${s}_$tag -f python tools/eval_bench.py $s > $out/ncu_eval_${s}_$tag.txt 2>&1
done
fi
