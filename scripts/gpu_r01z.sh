# Round-1 final evidence: bench N=1/2/4, reference arm, config-5 sweep at p=2/4, smoke.
export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01z
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01z/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r01z/bench_n1.log 2>&1; echo "bench n1 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01z/bench_reference_n1.log 2>&1; echo "ref rc=$?"
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2975$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench.py --gpus $NP > gpurun_out/r01z/bench_n$NP.log 2>&1; echo "bench n$NP rc=$?"
CUDA_VISIBLE_DEVICES=$CV timeout 1500 $TR bench_sweep.py --out gpurun_out/r01z/sweep_p$NP.jsonl > gpurun_out/r01z/sweep_p$NP.log 2>&1; echo "sweep p$NP rc=$?"
done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01z/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01z/launches_n1.csv $CMD > gpurun_out/r01z/ncu_list.log 2>&1; echo "ncu list rc=$?"
