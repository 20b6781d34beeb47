for d in 1 2 3; do
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c2 --depth $d 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('depth',$d,d['ray_bounces_per_step'],d['stage_ms']['launch'],d['roofline']['nodes_per_bounce'],d['roofline']['tris_per_bounce'])"
done
