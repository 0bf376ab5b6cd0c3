set -x
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python tools/record_profile.py spectral > gpurun_out/smtime_r02e.csv 2>&1
python tools/smtime.py gpurun_out/smtime_r02e.csv gpurun_out/smtime_r02e.json > gpurun_out/smtime_r02e.txt
python - <<'PY'
import json
d=json.load(open('gpurun_out/smtime_r02e.json')); d['source']='profiles/smtime_r02e.csv'
json.dump(d,open('profiles/smtime_spectral_latest.json','w'),indent=1)
PY
python bench.py > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err
for s in 6 10 12; do python bench.py --no-cpu-baseline --no-legs --no-e2e --streams $s 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams', $s, round(d['value'],2))" >> gpurun_out/streams_r02e.txt; done
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-legs --no-e2e > gpurun_out/launches_r02e.csv 2>&1
