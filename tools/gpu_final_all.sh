# Round-end battery: GPU tests, smoke, then tools/gpu_final.sh (bench both arms, sweep, launches, ncu)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" 2>&1 | tail -1
# Round-end measurement battery (one gpurun call): bench (both arms), the
# c1-c5 sweep, ncu launch list of a short bench, ncu --set full captures of
# both vote kernels.  Outputs under gpurun_out/final_*.
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
timeout 900 python tools/sweep.py > gpurun_out/final_sweep.json 2> gpurun_out/final_sweep.err; echo "sweep rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-sharded \
  --no-cpu-baseline > gpurun_out/final_ncu_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote_kernel -s 1 -c 1 \
  -o gpurun_out/final_vote_c2 python tools/prof_vote.py c2 29791 > /dev/null 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote_blocks -s 1 -c 1 \
  -o gpurun_out/final_blocks_c4 python tools/prof_vote.py c4 9261 > /dev/null 2>&1; echo "ncu c4 rc=$?"
