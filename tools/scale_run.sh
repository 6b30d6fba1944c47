#!/bin/bash
# Multi-GPU runs for a box with several B200s (one process per GPU, torchrun, 127.0.0.1):
# the bench line at N = 1, 2, 4, 8 (headline = Hotspot2D replicas; configs.hotspot3d_large = the
# axis-0 slab strong-scaling run with the in-graph peer exchange) and the distributed parity tests.
# This round's boxes had one GPU; on those, ranks share it (protocol check only).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/scale
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4 8; do
  [ "$N" -gt "$NG" ] && [ "$N" -gt 1 ] && { echo "skip N=$N (box has $NG GPUs)"; continue; }
  if [ "$N" = 1 ]; then
    python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/scale/bench_n1.json 2> gpurun_out/scale/bench_n1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --gpus $N --steps 5 --warmup 3 \
      > gpurun_out/scale/bench_n$N.json 2> gpurun_out/scale/bench_n$N.err
  fi
  echo "N=$N rc=$?"
  python -c "
import json; d = json.loads(open('gpurun_out/scale/bench_n$N.json').readline())
c = d['configs'].get('hotspot3d_large', {})
print('N=$N', 'headline', d['value'], d['unit'], '| hotspot3d_large us/iter', c.get('us_per_iter'), 'HBM frac per GPU', c.get('roofline', {}).get('frac'))"
done
