export TC_TIMEOUT_MS=20000
NP=${NP:-2}
mkdir -p gpurun_out/r01
timeout 900 python -m pytest tests/test_gpu_esgd.py -x -q 2>&1 | tail -2
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29518 bench_sweep.py --out gpurun_out/r01/sweep_p$NP.jsonl > gpurun_out/r01/sweep_p$NP.log 2>&1; echo "sweep rc=$?"
tail -3 gpurun_out/r01/sweep_p$NP.log
