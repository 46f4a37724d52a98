# f1 on a real ResNet-50 backward pass, iterations captured as CUDA graphs, modes interleaved
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() { N=$1; shift; CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2971$N bench_train.py "$@" 2>>gpurun_out/train_graph2.err | grep '{' | tee -a gpurun_out/train_graph2.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['bucket_mb'], d['ctas'], d['mode'], d['side_stream_priority'], 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'step', round(d['t_step_alone_us']), 'hidden', round(d['hidden_fraction'],2), d['replicas_identical'], d['rounds']['overlap'])"; }
run 4 --graph --channels-last
run 4 --graph --channels-last --priority
run 4 --graph --channels-last --priority --ctas 64
run 4 --graph --channels-last --priority --bucket-mb 64
run 4 --graph --channels-last --priority --split --ctas 32
run 4 --graph --channels-last --priority --split
run 2 --graph --channels-last --priority
run 2 --graph --channels-last
