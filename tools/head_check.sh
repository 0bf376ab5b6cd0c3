# Validate HEAD on a fresh box: the GPU suite, smoke(), one default bench line.
set -x
tag=${1:-r02h}
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$tag.log 2>&1; echo rc=$? >> gpurun_out/gputest_$tag.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$tag.log 2>&1
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
