# cross3m bulk-copy (TMA) variant: parity of the spectral covariance tests, then an A/B against
# the cp.async kernel (-DSSI_CROSS_CPASYNC=1) on the c3 covariance call and on the c3 bench.
set -x
python -m paper_2411_05510_b200.build --force > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "spectral" > gpurun_out/cross_tma_parity.log 2>&1; echo rc=$? >> gpurun_out/cross_tma_parity.log
python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/cross_tma_fullsize.log 2>&1; echo rc=$? >> gpurun_out/cross_tma_fullsize.log
bash tools/cov_ab.sh "" "-DSSI_CROSS_CPASYNC=1" "" "-DSSI_CROSS_CPASYNC=1" > gpurun_out/cross_tma_cov_ab.txt 2>&1
bash tools/knob_ab.sh "" "-DSSI_CROSS_CPASYNC=1" > gpurun_out/cross_tma_bench_ab.txt 2>&1
python -m paper_2411_05510_b200.build --force > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:cross3m -s 2 -c 1 -o gpurun_out/cross3m_tma_r02 python tools/cov_only.py c3 spectral > gpurun_out/cross_tma_ncu.log 2>&1
