export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2952$NP"
timeout 600 $TR bench_sweep.py --sizes 0,1,2,3,4,5,6 --tensors 1,32,161 --out gpurun_out/r01/sweep_ll2_p${NP}.jsonl > /dev/null 2>&1; echo "p$NP rc=$?"
done
