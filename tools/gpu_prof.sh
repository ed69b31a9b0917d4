# ncu --set full of the vote kernel on a c2 slice (after a plain run of the same command)
mkdir -p gpurun_out
CFG=${1:-c2}; NR=${2:-4096}; TAG=${3:-vote}
timeout 300 python tools/prof_vote.py $CFG $NR > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vote_kernel -s 1 -c 1 -o gpurun_out/${TAG}_${CFG} python tools/prof_vote.py $CFG $NR > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
