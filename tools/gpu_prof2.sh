# ncu --set full of the vote kernel for two configs (after plain runs)
mkdir -p gpurun_out
for spec in "$@"; do
  CFG=${spec%%:*}; NR=${spec##*:}
  timeout 300 python tools/prof_vote.py $CFG $NR > gpurun_out/prof_plain_$CFG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:vote_kernel -s 1 -c 1 -o gpurun_out/${TAG}_${CFG} python tools/prof_vote.py $CFG $NR > gpurun_out/ncu_full_$CFG.log 2>&1; echo "ncu $CFG rc=$?"
done
