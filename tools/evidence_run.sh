set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02f.log 2>&1; echo rc=$? >> gpurun_out/gputest_r02f.log
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python tools/record_profile.py spectral > gpurun_out/smtime_r02f.csv 2>&1
python tools/smtime.py gpurun_out/smtime_r02f.csv gpurun_out/smtime_r02f.json > gpurun_out/smtime_r02f.txt
python - <<'PY'
import json
d=json.load(open('gpurun_out/smtime_r02f.json')); d['source']='profiles/smtime_r02f.csv'
json.dump(d,open('profiles/smtime_spectral_latest.json','w'),indent=1)
PY
python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-legs --no-e2e > gpurun_out/launches_r02f.csv 2>&1
