# bench.py with NVLS (algorithm 4) as the timed step at N = 4 and 3: the code path the automatic choice takes from N = 5
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
for N in 4 3; do
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2957$N bench.py --gpus $N --algo 4 > gpurun_out/nvbench_n$N.json 2> gpurun_out/nvbench_n$N.err; echo "rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/nvbench_n$N.json') if l.startswith('{')][-1])
print($N, round(d['t_us'],1), d['launch'], json.dumps(d['roofline'])[:300], d['clocks'])"
done
