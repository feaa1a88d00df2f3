export RCV_TIMEOUT_S=3
for NUMEL in 118592 1185920 12441600 124439808; do
  echo "== numel $NUMEL"
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 tools/gate_debug.py $NUMEL 6 4 2>&1 | grep "^rank\|Error" | head -20
done
