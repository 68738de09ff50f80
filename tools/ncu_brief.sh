#!/bin/bash
# Key counters of every kernel in an .ncu-rep (run here, no GPU needed).
for f in "$@"; do
  echo "== $f"
  ncu -i "$f" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]
want=['Kernel Name','gpu__time_duration.sum','sm__cycles_elapsed.avg.per_second','dram__bytes_read.sum','dram__bytes_write.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active','lts__t_sectors_srcunit_tex_op_read.sum','lts__t_sectors_srcunit_tex_op_write.sum','smsp__inst_executed.sum','launch__grid_size','launch__registers_per_thread']
for row in r[2:]:
  print('  '.join(f'{w.split(\".\")[0]}={row[h.index(w)]}{r[1][h.index(w)]}' for w in want if w in h))
"
done
