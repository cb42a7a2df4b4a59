mkdir -p gpurun_out/s4v
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/s4v/pytest.log 2>&1; echo "rc $?" >> gpurun_out/s4v/pytest.log
