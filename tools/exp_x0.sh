timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
PIT_X0=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
python tools/trace_run.py 2 4 5
PIT_X0=1 python tools/trace_run.py 2 3 4 5
