mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coupled.py -x -q -m gpu > gpurun_out/coupled_tests.log 2>&1; echo ctests=$?
tail -15 gpurun_out/coupled_tests.log
