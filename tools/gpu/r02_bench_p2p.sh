# bench lines at N = 2, 4 with the same-run P2P pull ceiling in the roofline object
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2953$N bench.py --gpus $N > gpurun_out/bench_p2p_n$N.json 2> gpurun_out/bench_p2p_n$N.err; echo "bench$N rc=$?"
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_p2p_n$N.json') if l.startswith('{')][-1])
r=d['roofline']; print($N, round(d['t_us'],1), round(r['achieved']), r.get('frac_of_p2p_pull_peak'), json.dumps(r.get('p2p_pull_peak'))[:400])"
done
