#!/bin/bash
# A/B the library variants built by tools/variants.py on the default bench workload.
# usage: tools/ab.sh name1 name2 ...   (name "base" = libb200rt.so)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then lib=libb200rt.so; else lib=libb200rt_$v.so; fi
  timeout 600 python tools/ab_run.py $lib bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-c2 \
    > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "$v rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);print(round(d['value']/1e9,3),'Gbounce/s', d['stage_ms'])" 2>&1 | tail -1)"
done
