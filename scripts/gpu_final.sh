export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/rfinal
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rfinal/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rfinal/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/rfinal/bench_n1.log 2>&1; echo "bench n1 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rfinal/bench_reference_n1.log 2>&1; echo "ref rc=$?"
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2981$NP bench.py --gpus $NP > gpurun_out/rfinal/bench_n$NP.log 2>&1; echo "bench n$NP rc=$?"
done
