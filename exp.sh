summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9,3), d['stage_ms']['launch'], d['stage_ms']['validate'], round(d['roofline']['nodes_per_bounce'],2), round(d['roofline']['tris_per_bounce'],2))"; }
timeout 300 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -1
B200RT_LIB=libb200rt_w4.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "launch or intersect or coverage" 2>&1 | tail -1
echo binary; timeout 300 python bench.py --no-cpu --no-e2e --no-c2 --steps 3 2>&1 | summ
echo wide4; B200RT_LIB=libb200rt_w4.so timeout 300 python bench.py --no-cpu --no-e2e --no-c2 --steps 3 2>&1 | summ
