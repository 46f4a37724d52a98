# final round-1 bench lines on the HEAD build: N = 1 (+ reference arm), 2, 4
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo n1 $?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref_n1.json 2> gpurun_out/final_ref_n1.err; echo ref $?
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err; echo n$N $?
done
