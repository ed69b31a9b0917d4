# quick A/B round: gpu tests + per-config vote timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in c1 c2 c3 c4 c2local c2l2; do timeout 300 python tools/variant_time.py $c; done
