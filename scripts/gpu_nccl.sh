#!/bin/bash
# The bench's torchrun path (NCCL process group, multiview.render_path) on the one GPU a
# gpurun box has: N=1 under torch.distributed.run, configs 3 and 5, NCCL_DEBUG=INFO.
set -u
OUT=gpurun_out
mkdir -p $OUT
for cfg in 3 5; do
  NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
    --master-addr 127.0.0.1 --master-port 2951$cfg bench.py --gpus 1 --steps 50 --warmup 5 --config $cfg --no-cpu --no-cub \
    > $OUT/nccl_c$cfg.json 2> $OUT/nccl_c$cfg.err; echo "torchrun config $cfg rc=$?"
  grep '^{' $OUT/nccl_c$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'gather', json.dumps(d.get('gather'))[:400])"
  grep -m3 "NCCL INFO.*\(version\|Init COMPLETE\|comm\)" $OUT/nccl_c$cfg.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_arm.json 2> $OUT/ref_arm.err; echo "reference arm rc=$?"; tail -c 600 $OUT/ref_arm.json
