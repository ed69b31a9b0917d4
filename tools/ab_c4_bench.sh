# bench.py c4 e2e legs against alternative builds (DSES_LIB)
for lib in "$@"; do
  DSES_LIB=$lib timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-sharded --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print('$lib', 'value %.3g' % d['value'], 'batch %.3g' % e['value'], 'single %.3g' % e['single_call']['value'])"
done
