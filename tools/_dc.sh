mkdir -p gpurun_out/s4s
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4s/pytest.log 2>&1; echo "rc $?" >> gpurun_out/s4s/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4s/smoke.log 2>&1; echo "rc $?" >> gpurun_out/s4s/smoke.log
timeout 600 python bench.py > gpurun_out/s4s/bench.json 2> gpurun_out/s4s/bench.err; echo "rc $?" >> gpurun_out/s4s/bench.err
