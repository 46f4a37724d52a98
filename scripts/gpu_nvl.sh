export TC_TIMEOUT_MS=20000
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 2 --steps 100 --no-e2e > /tmp/n2.log 2>&1; echo rc=$?
tail -5 /tmp/n2.log | cut -c1-600
python - <<'PY'
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
v = nv.nvmlDeviceGetFieldValues(h, [138, 139])
for x in v: print(x.fieldId, x.nvmlReturn, x.value.ullVal, x.scopeId)
PY
