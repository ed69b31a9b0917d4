# A/B timing of the built library variants in paper_2502_00115_b200/_lib/ on c2 and c4
for v in paper_2502_00115_b200/_lib/libdses_b200*.so; do for c in ${CFGS:-c2 c4}; do timeout 300 python tools/variant_time.py $c $PWD/$v; done; done
