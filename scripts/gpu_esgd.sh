export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01g
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 > gpurun_out/r01g/bench_n1.log 2>&1; echo "bench n1 rc=$?"
tail -1 gpurun_out/r01g/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1', d['t_us'], d['easgd'], d['esgd_fused'])"
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2962$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench.py --gpus $NP --steps 100 --no-e2e > gpurun_out/r01g/bench_n$NP.log 2>&1; echo "bench n$NP rc=$?"
tail -1 gpurun_out/r01g/bench_n$NP.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$NP', d['t_us'], d['easgd'], d['esgd_fused'])"
done
