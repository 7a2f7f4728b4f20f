timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout 900 python tools/c3_certificate.py gpurun_out/r02_c3_certificate.json > gpurun_out/c3cert.log 2>&1; tail -3 gpurun_out/c3cert.log
