set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02g.log 2>&1; echo rc=$? >> gpurun_out/gputest_r02g.log
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python tools/record_profile.py spectral > gpurun_out/smtime_r02g.csv 2>&1
python tools/smtime.py gpurun_out/smtime_r02g.csv gpurun_out/smtime_r02g.json > gpurun_out/smtime_r02g.txt
python - <<'PY'
import json
d=json.load(open('gpurun_out/smtime_r02g.json')); d['source']='profiles/smtime_r02g.csv'
json.dump(d,open('profiles/smtime_spectral_latest.json','w'),indent=1)
PY
python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-legs --no-e2e > gpurun_out/launches_r02g.csv 2>&1
python tools/sweep_projection.py gpurun_out/sweep_projection_r02g.json > gpurun_out/sweep_projection_r02g.txt 2>&1
for a in "--steps 20 --warmup 5" "--steps 20 --warmup 5"; do python bench.py $a --no-cpu-baseline --no-legs 2>/dev/null | tail -1 > /tmp/k.json; python -c "import json; d=json.load(open(\"/tmp/k.json\")); print(\"$a\", round(d[\"value\"],2), round(d[\"e2e\"][\"value\"],2))" >> gpurun_out/k20_r02g.txt; done
