export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01h
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2966$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 900 $TR bench_sweep.py --sizes 7,8,9 --tensors 1,161,1024 --out gpurun_out/r01h/sweep_p$NP.jsonl > /dev/null 2>&1; echo "sweep p$NP rc=$?"
done
