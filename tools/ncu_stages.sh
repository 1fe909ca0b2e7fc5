#!/bin/bash
# ncu evidence for every kernel of one config-4 pool step (duration + DRAM
# bytes per launch) and a --set full capture of the config-5 sweep kernel.
# Run on the GPU box: tools/gpu.sh 'bash tools/ncu_stages.sh <tag>'
set -x
TAG=${1:-r2}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/${TAG}_config4_dram.csv \
  python tools/stage_probe.py --reps 1 > gpurun_out/${TAG}_config4_probe.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_sweep -c 1 \
  -o gpurun_out/${TAG}_sweep_full python tools/sweep_probe.py 1 > gpurun_out/${TAG}_sweep_ncu.log 2>&1
timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/${TAG}_sweep_dram.csv python tools/sweep_probe.py 2 \
  > /dev/null 2>&1
true
