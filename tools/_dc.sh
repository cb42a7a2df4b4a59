mkdir -p gpurun_out/s4x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4x/pytest.log 2>&1; echo "rc $?" >> gpurun_out/s4x/pytest.log
timeout 120 python tools/diag_configs.py > gpurun_out/s4x/configs.txt 2>&1
