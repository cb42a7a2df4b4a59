mkdir -p gpurun_out/s4f
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4f/pytest.log 2>&1; echo "rc $?" >> gpurun_out/s4f/pytest.log
timeout 600 python tools/dense_check.py > gpurun_out/s4f/dc.txt 2>&1
timeout 300 python tools/diag_configs.py > gpurun_out/s4f/configs.txt 2>&1
nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/s4f/configs.txt
