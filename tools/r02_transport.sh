#!/bin/bash
# world-1 multi-GPU path (--partition) with each exchange transport: the
# per-iteration cost of the captured exchange (NCCL all-gather vs
# peer-memory stores + flags).  Results in gpurun_out/r02_transport_*.json.
set -u
mkdir -p gpurun_out
for w in pack5000 mpc100k svm1m; do
  for t in nccl p2p; do
    extra=""; [ "$w" = svm1m ] && extra="--points-per-rank 1000000"
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
        --master-port 29533 bench.py --partition --workload $w --transport $t --steps 200 --warmup 5 $extra \
        > gpurun_out/r02_transport_${w}_$t.json 2> gpurun_out/r02_transport_${w}_$t.err
    echo "$w $t rc=$?"; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['config']['parallelism'])" gpurun_out/r02_transport_${w}_$t.json
  done
done
