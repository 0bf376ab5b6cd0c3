# Launch list (ncu, per-launch durations + SM-active cycles) of the bench command and the one-record
# SM-time table at HEAD; then three driver-length bench runs. Usage: bash tools/launches_head.sh TAG
set -x
tag=${1:-r02j}
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python tools/record_profile.py spectral > gpurun_out/smtime_$tag.csv 2>&1
python tools/smtime.py gpurun_out/smtime_$tag.csv gpurun_out/smtime_$tag.json > gpurun_out/smtime_$tag.txt
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none -c 3000 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-legs --no-e2e > gpurun_out/launches_$tag.csv 2>&1
for r in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-legs 2>/dev/null | tail -1 > gpurun_out/bench_k20_${tag}_$r.json; done
