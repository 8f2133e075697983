#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line (+ reference arm), launch list,
# ncu --set full on the top kernels.   usage: tools/gpu_check.sh TAG [ncu-kernel-regex] [skip] [count]
TAG=${1:-check}
KRE=${2:-'raster_bwd_tile1w|raster_bwd_kernel|ssim_loss_kernel|pcols_fwd|pcols_bwd|raster_fwd_kernel|srows_inv|srows_fwd|adan_fused|scatter_ids'}
SKIP=${3:-22}; CNT=${4:-11}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.jsonl 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py cfg2 4 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s ${SKIP} -c ${CNT} \
   -o gpurun_out/${TAG}_full -f python tools/profile_step.py cfg2 4 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_smoke.log
cut -c1-300 gpurun_out/${TAG}_bench.jsonl
cut -c1-300 gpurun_out/${TAG}_bench_ref.jsonl
