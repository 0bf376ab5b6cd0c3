python -m pytest tests/test_gpu_e3.py tests/test_gpu_parity.py -x -q -k "e3 or rsvd" > gpurun_out/e3d_pytest.log 2>&1; echo pytest=$? >> gpurun_out/e3d_pytest.log
SSI_CHOL_PROFILE=1 python tools/e3_rsvd_only.py > gpurun_out/e3d_cholprof.log 2>&1
python tools/e3_time.py > gpurun_out/e3d_time.json 2> gpurun_out/e3d_time.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e3d_launches.csv python tools/e3_rsvd_only.py > gpurun_out/e3d_ncu.log 2>&1
