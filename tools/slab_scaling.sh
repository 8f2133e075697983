#!/bin/bash
# Row-slab decomposition on ONE GPU: work per rank (ms) for R virtual ranks
# (peer-put exchange; no interconnect time).  usage: tools/slab_scaling.sh > out.md
echo "| workload | R | ms per rank (R ranks on one GPU / R) | unsharded graph step (ms) |"
echo "|---|---|---|---|"
for w in ${WORKLOADS:-cfg2 cfg3 cfg4}; do
  base=$(timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;print(round(json.loads(sys.stdin.read())['ms_per_step'],3))")
  for R in 1 2 4 8; do
    if [ $R -eq 1 ]; then a="--shard slabs --steps 10 --warmup 3"; else a="--shard slabs --virtual-ranks $R --steps 10 --warmup 3"; fi
    ms=$(timeout 600 python bench.py --workload $w $a 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());v=d.get('virtual_ranks');print(round(v['ms_per_rank_compute'] if v else d['ms_per_step'],3))")
    echo "| $w | $R | $ms | $base |"
  done
done
