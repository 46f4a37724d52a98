timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo tests $? >> gpurun_out/gpu_tests4.log
for N in 4 3; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench$N $?; done
