# Build kernel variants (extra -D flags) as separate libraries under variants/ for A/B timing:
#   bash tools/build_variants.sh name1 "-DFOO=1" name2 "-DBAR" ...
# then on the GPU: LC_B200_LIB=variants/name1.so python bench.py --no-cpu-baseline
set -e
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -lineinfo -std=c++17 -shared -Xcompiler -fPIC $flags \
    -o variants/$name.so paper_2601_06288_b200/csrc/llmconf_b200.cu &
done
wait
ls -la variants
