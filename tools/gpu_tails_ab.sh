# K3 A/B: GPU tests on the in-tree library, then bench kernel times for every variants/*.so
#   bash tools/gpu_tails_ab.sh <tag>
mkdir -p gpurun_out
tag=${1:-tails}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_${tag}.log
bash tools/gpu_variants.sh
