# End-of-session evidence at HEAD: GPU suite, smoke, default bench, two driver-length bench runs.
set -x
tag=${1:-r02i}
python -m pytest tests -m gpu -q > gpurun_out/gputest_$tag.log 2>&1; echo rc=$? >> gpurun_out/gputest_$tag.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$tag.log 2>&1
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
for r in 1 2; do python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/bench_k20_${tag}_$r.json; done
