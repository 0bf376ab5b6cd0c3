# cross3m bulk-copy variant 2 (last-warp refill): parity, then A/B against the default cp.async kernel.
set -x
SSI_NVCC_EXTRA="-DSSI_CROSS_TMA=2" python -m paper_2411_05510_b200.build --force > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "spectral" > gpurun_out/cross_tma2_parity.log 2>&1; echo rc=$? >> gpurun_out/cross_tma2_parity.log
python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/cross_tma2_fullsize.log 2>&1; echo rc=$? >> gpurun_out/cross_tma2_fullsize.log
bash tools/cov_ab.sh "" "-DSSI_CROSS_TMA=2" "" "-DSSI_CROSS_TMA=2" > gpurun_out/cross_tma2_cov_ab.txt 2>&1
bash tools/knob_ab.sh "" "-DSSI_CROSS_TMA=2" > gpurun_out/cross_tma2_bench_ab.txt 2>&1
