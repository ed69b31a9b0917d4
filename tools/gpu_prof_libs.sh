# ncu --set full of the vote kernel for several libraries on one config slice:
# LIBS="a.so b.so" CFG=c2 NR=4096 TAG=x bash tools/gpu_prof_libs.sh
mkdir -p gpurun_out
for v in ${LIBS}; do
  n=$(basename $v .so)
  DSES_LIB=$PWD/$v timeout 300 python tools/prof_vote.py ${CFG:-c2} ${NR:-4096} > /dev/null 2>&1 && \
  DSES_LIB=$PWD/$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:vote_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG:-cmp}_${n}_${CFG:-c2} python tools/prof_vote.py ${CFG:-c2} ${NR:-4096} > /dev/null 2>&1; echo "ncu $n rc=$?"
done
