# A/B of the pipeline's tail hint at the driver's 20 steps and at 80 (alternating). bash tools/tail_ab.sh
out=gpurun_out/tail_ab.txt; : > $out
for rep in 1 2; do for t in 0 1 2 4 7; do for a in "--steps 20 --warmup 5" "--steps 80 --warmup 8"; do
  python bench.py $a --tail $t --no-cpu-baseline --no-legs 2>/dev/null | tail -1 > /tmp/k.json
  python -c "import json; d=json.load(open('/tmp/k.json')); print('tail $t $a', round(d['value'],2), round(d['e2e']['value'],2))" >> $out
done; done; done
cat $out
