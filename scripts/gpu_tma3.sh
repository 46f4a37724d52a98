export TC_TIMEOUT_MS=10000
mkdir -p gpurun_out/r01
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --steps 200 --warmup 10 2>/dev/null | tail -1 > gpurun_out/r01/bench_n1_tma.json
python -c "import json,sys; d=json.load(open('gpurun_out/r01/bench_n1_tma.json')); print('N1', round(d['t_us'],1), round(d['roofline']['frac'],3), d['easgd']['t_us'], d['e2e'], d['clocks'])"
done
