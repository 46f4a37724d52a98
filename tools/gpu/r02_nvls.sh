# NVLS iteration: real-process parity (p = 2, 4) and per-algorithm timings at p = 4
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/mp_nvls.log 2>&1; echo "mp rc=$?"
timeout 300 $TR --nproc-per-node 4 --master-port 29571 tools/algo_bench.py --algos 6,4 > gpurun_out/algo_p4.jsonl 2> gpurun_out/algo_p4.err; echo "algo4 rc=$?"
cat gpurun_out/algo_p4.jsonl
