timeout 900 python -m pytest tests/test_gpu_cli.py -x -q > gpurun_out/pytest_cli.log 2>&1; echo pytest=$?
