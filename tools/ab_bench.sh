#!/bin/bash
# A/B of the current tree against an older tree ($AB_OLD, e.g. a `git archive` of a previous
# commit) on one box: the same bench command, alternated, twice each.
set -x
R=$GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 8 --no-cpu-baseline --no-legs --no-e2e"
python -m paper_2411_05510_b200.build --force > gpurun_out/ab_build.log 2>&1
(cd $AB_OLD && python -m paper_2411_05510_b200.build --force > /dev/null 2>&1)
for r in 1 2; do
  $B > gpurun_out/ab_cur_$r.json 2>>gpurun_out/ab.err
  (cd $AB_OLD && python bench.py --steps 40 --warmup 8 --no-cpu-baseline --no-e2e > $R/gpurun_out/ab_old_$r.json 2>>$R/gpurun_out/ab.err)
done
