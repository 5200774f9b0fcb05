# A/B: bench every variants/*.so (kernel-only config5 numbers), then the GPU tests on the in-tree build.
#   bash tools/gpu_ab.sh [pytest args]
mkdir -p gpurun_out
bash tools/gpu_variants.sh
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
  tail -4 gpurun_out/pytest_gpu.log
fi
