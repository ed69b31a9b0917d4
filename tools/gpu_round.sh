# Full GPU round: tests, smoke, bench (both arms), launch list, ncu full capture of the vote kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
cat gpurun_out/bench_ref.json
# launch list of the same bench command (device-resident steps only, no CPU baseline)
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sharded > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sharded > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
# the bench's vote launch: c2 seed-0 pair, all 29,791 rotations
timeout 300 python tools/prof_vote.py c2 29791 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:vote_kernel -s 1 -c 1 -o gpurun_out/vote_full python tools/prof_vote.py c2 29791 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
