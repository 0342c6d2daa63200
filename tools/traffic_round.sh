#!/bin/bash
# DRAM traffic per packet of every bench config (run on the GPU box from the
# repo root): one ncu launch list with the DRAM counters per config /
# precision, reduced by tools/packet_traffic.py into gpurun_out/traffic/.
set -u
O=gpurun_out/traffic
mkdir -p $O
for c in C1 C2 C3 C4 C5; do for p in f64 f32; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv -c 300 --log-file $O/launches_${c}_$p.csv \
      python bench.py --config $c --precision $p --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python tools/packet_traffic.py $O/launches_${c}_$p.csv > $O/packet_${c}_$p.txt 2>&1
done; done
ls -la $O
