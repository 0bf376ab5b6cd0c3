#!/bin/bash
# A/B of compile-time knobs on the headline: for each SSI_NVCC_EXTRA value (arguments; "" =
# default) rebuild libssi and run the c3 bench (device records/s, no legs / e2e / CPU leg);
# the variants alternate, two rounds (AB AB), so box drift hits every variant alike.
for r in 1 2; do
  for v in "$@"; do
    SSI_NVCC_EXTRA="$v" python -m paper_2411_05510_b200.build --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
    python bench.py --steps 40 --warmup 8 --no-cpu-baseline --no-legs --no-e2e 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('[$v]', round(d['value'], 2), 'rec/s', round(d['ms_per_step'], 3), 'ms', d['clocks']['reasons'])"
  done
done
SSI_NVCC_EXTRA="" python -m paper_2411_05510_b200.build --force > /dev/null 2>&1
