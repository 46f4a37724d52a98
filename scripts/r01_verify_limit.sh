# after the p = 4 one-shot limit change: GPU suite, the p = 4 sweep at 1/4/16 MiB, bench N = 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_v.log 2>&1; echo tests $?
TR="timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
$TR --nproc-per-node 4 bench_sweep.py --sizes 5,6,7 > gpurun_out/os_auto_new_p4.jsonl 2>/dev/null; echo sweep $?
$TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/bench_v_n4.json 2>gpurun_out/bench_v_n4.err; echo bench4 $?
