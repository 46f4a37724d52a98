export TC_TIMEOUT_MS=10000
timeout 300 python tools/local_variants.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1', round(d['t_us'],1), round(d['roofline']['frac'],3), d['easgd'])"
