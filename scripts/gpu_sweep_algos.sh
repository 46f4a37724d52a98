export TC_TIMEOUT_MS=20000
NP=${NP:-4}
mkdir -p gpurun_out/r01
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29520"
for cfg in "1 0" "3 0" "0 8388608"; do
  set -- $cfg
  timeout 600 $TR bench_sweep.py --algo $1 --oneshot $2 --sizes 5,6,7,8,9 --tensors 1,161 --out gpurun_out/r01/sweep_p${NP}_a$1_o$2.jsonl > /dev/null 2>&1; echo "algo $1 oneshot $2 rc=$?"
done
