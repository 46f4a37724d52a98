export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01j
for C in alexnet vgg16; do
timeout 600 python bench.py --config $C --steps 50 --no-cpu-baseline > gpurun_out/r01j/bench_${C}_n1.log 2>&1; echo "$C n1 rc=$?"
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2970$NP bench.py --gpus $NP --config $C --steps 50 > gpurun_out/r01j/bench_${C}_n$NP.log 2>&1; echo "$C n$NP rc=$?"
done
done
