mkdir -p gpurun_out
GNSB_DEBUG=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -60 > gpurun_out/pytest_debug.log
