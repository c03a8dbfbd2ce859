#!/bin/bash
# k_zx row-chunk sweep at config 5: ncu duration of k_zx per AXB_Z_JROWS
for jr in 32 64 128 256 512; do
  t=$(AXB_Z_JROWS=$jr timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_zx -s 3 -c 2 python bench.py --config 5 --steps 3 --warmup 3 2>/dev/null | grep duration | awk '{print $3}' | tr '\n' ' ')
  echo "jrows=$jr k_zx_us: $t"
done
