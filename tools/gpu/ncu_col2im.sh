mkdir -p gpurun_out/tmp
timeout 300 python tools/ncu_step.py alexconv_b128 2 > gpurun_out/col2im_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"col2im|premove" -s 10 -c 4 -f -o gpurun_out/tmp/c2i python tools/ncu_step.py alexconv_b128 2 > gpurun_out/col2im_ncu.log 2>&1; echo "ncu $?"
python tools/ncu_summary.py gpurun_out/tmp/c2i.ncu-rep > gpurun_out/r2_ncu_col2im_summary.txt 2>&1; cat gpurun_out/r2_ncu_col2im_summary.txt | head -60
python tools/ncu_stalls.py gpurun_out/tmp/c2i.ncu-rep 25 > gpurun_out/r2_ncu_col2im_stalls.txt 2>&1; head -30 gpurun_out/r2_ncu_col2im_stalls.txt
ncu -i gpurun_out/tmp/c2i.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers','smsp__average_warp_latency_issue_stalled_long_scoreboard','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct']
ix=[h.index(w) for w in want if w in h]
for row in r[2:]: print(' | '.join(h[i].split('__')[-1][:40]+'='+row[i][:40] for i in ix))
" > gpurun_out/r2_ncu_col2im_raw.txt; cat gpurun_out/r2_ncu_col2im_raw.txt
rm -rf gpurun_out/tmp
