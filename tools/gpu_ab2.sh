# A/B round: gpu tests, then per-config vote timings of the current library vs libdses_v1.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in ${CFGS:-c1 c2 c4 c2local}; do
  timeout 300 python tools/variant_time.py $c
  [ -f paper_2502_00115_b200/_lib/libdses_v1.so ] && timeout 300 python tools/variant_time.py $c $PWD/paper_2502_00115_b200/_lib/libdses_v1.so
done
