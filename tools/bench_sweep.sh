for a in "--streams 8" "--streams 10" "--streams 12" "--streams 6" "--streams 8 --no-priority"; do
  python bench.py --no-cpu-baseline $a > gpurun_out/bs.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bs.json').read().strip().splitlines()[-1]); print('$a', round(d['value'],2), round(d['e2e']['value'],2))"
done
