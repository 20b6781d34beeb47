for v in base s8 s12; do
  if [ "$v" = base ]; then lib=libb200rt.so; else lib=libb200rt_$v.so; fi
  echo "== $v"; python tools/ab_run.py $lib tools/build_profile.py | tail -2
  python tools/ab_run.py $lib bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-c2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['stage_ms']['launch'], d['roofline']['nodes_per_bounce'])"
done
