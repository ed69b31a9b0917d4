# vote/search timing of several built libraries: LIBS="a.so b.so" CFGS="c2 c4"
mkdir -p gpurun_out
for v in ${LIBS}; do for c in ${CFGS:-c2 c4}; do echo -n "$(basename $v) "; timeout 300 python tools/variant_time.py $c $PWD/$v | cut -c1-150; done; done
