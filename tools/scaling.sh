#!/bin/bash
# Weak-scaling run of the bench contract at 1, 2, ..., $MAXG GPUs (one process
# per GPU via torchrun for N > 1), then the alpha-beta model comparison at $MAXG.
export PYTHONPATH=.
MAXG=${MAXG:-4}
ARGS=${ARGS:-"--steps 3 --warmup 3 --no-cpu-baseline"}
g=1
while [ $g -le $MAXG ]; do
  if [ $g -eq 1 ]; then
    timeout 600 python bench.py --gpus 1 $ARGS > gpurun_out/scale_g1.json 2> gpurun_out/scale_g1.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 \
      --master-port $((29600 + g)) bench.py --gpus $g $ARGS > gpurun_out/scale_g$g.json 2> gpurun_out/scale_g$g.err
  fi
  g=$((g * 2))
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $MAXG --master-addr 127.0.0.1 \
  --master-port 29650 tools/alpha_beta.py --out gpurun_out/alpha_beta_g$MAXG.json > gpurun_out/alpha_beta_g$MAXG.log 2>&1
