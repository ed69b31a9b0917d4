# k-d leaf fill sweep: vote/search timing per DSES_KD_FILL on c1..c4 + c2local
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or api" 2>&1 | tail -3
for f in ${FILLS:-1.0 0.97 0.94 0.90}; do
  for c in ${CFGS:-c2 c4 c2local c1}; do DSES_KD_FILL=$f timeout 300 python tools/variant_time.py $c; done
done
