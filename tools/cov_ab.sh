#!/bin/bash
# A/B of covariance-kernel compile-time variants on one box: for each SSI_NVCC_EXTRA value
# (arguments; "" = default) rebuild libssi and time the c3 covariance call twice.
for v in "$@"; do
  SSI_NVCC_EXTRA="$v" python -m paper_2411_05510_b200.build --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for r in 1 2; do SSI_NVCC_EXTRA="$v" python tools/cov_time.py c3 spectral; done
done
