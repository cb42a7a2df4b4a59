python -m pytest -q -x tests/test_gpu_configs.py::test_cfg2_batch1_many_inputs_within_bound tests/test_gpu_parity.py -k "batch1 or headline or swap or zero" 2>&1 | tail -1
python tools/diag_latency.py --batches 1 --reps 400 2>&1 | grep "flush=True"
python tools/b1_timeline.py --reps 1
