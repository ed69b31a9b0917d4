# GPU test suite against a bounds-checked build (device asserts on every
# histogram update / point index; compute-sanitizer is closed on the pool).
set -e
cd paper_2502_00115_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -DDSES_DEBUG_BOUNDS -o /tmp/libdses_b200_debug.so \
  csrc/dses_vote.cu csrc/dses_score.cu csrc/dses_sparse.cu csrc/dses_capi.cu csrc/dses_probe.cu
cd ..
DSES_LIB=/tmp/libdses_b200_debug.so python -m pytest tests -m gpu -q -x
