# Evidence after the TMA two-shot: bench N=1/2/4 and the config-5 sweep at p=2/4 (automatic choice).
export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01f
timeout 600 python bench.py > gpurun_out/r01f/bench_n1.log 2>&1; echo "bench n1 rc=$?"
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2961$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench.py --gpus $NP > gpurun_out/r01f/bench_n$NP.log 2>&1; echo "bench n$NP rc=$?"
CUDA_VISIBLE_DEVICES=$CV timeout 1200 $TR bench_sweep.py --tensors 1,32,161,1024 --out gpurun_out/r01f/sweep_p$NP.jsonl > gpurun_out/r01f/sweep_p$NP.log 2>&1; echo "sweep p$NP rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01f/bench_reference_n1.log 2>&1; echo "ref rc=$?"
