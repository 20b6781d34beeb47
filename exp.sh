summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9,3), d['stage_ms']['launch'], d['stage_ms']['validate'], round(d['roofline']['nodes_per_bounce'],2), round(d['roofline']['tris_per_bounce'],2))"; }
for v in "" $VARIANTS; do
  if [ -z "$v" ]; then lib=""; else lib="libb200rt_$v.so"; fi
  echo "variant ${v:-default}: $(B200RT_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --no-c2 --steps 3 2>&1 | summ)"
done
