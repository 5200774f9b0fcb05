mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.txt 2>&1; echo sharded rc=$?
tail -30 gpurun_out/pytest_sharded.txt
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_sharded.py > gpurun_out/pytest_gpu.txt 2>&1; echo gpu rc=$?
tail -3 gpurun_out/pytest_gpu.txt
