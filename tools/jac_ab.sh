for v in "" "-DSSI_JAC_STASYNC=1"; do
  SSI_NVCC_EXTRA="$v" python -m paper_2411_05510_b200.build --force > /dev/null 2>&1
  echo "[$v]"; SSI_JAC_PROFILE=1 timeout 300 python tools/rsvd_only.py 2>&1 | grep ring | head -1
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rsvd_toeplitz" 2>&1 | tail -1
done
python -m paper_2411_05510_b200.build --force > /dev/null 2>&1
