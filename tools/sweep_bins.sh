#!/bin/bash
# Binning diagnostics: per-kernel times of the config-3 precompute for several bucket counts.
P="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-cg"
for nb in ${@:-64 256 1024 4096}; do
  GSGPC_BIN_BUCKETS=$nb timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"k_partition|k_slice" -c 8 --csv --log-file gpurun_out/sweep_nb$nb.csv $P > /dev/null 2>&1
done
