import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
keys=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','lts__throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__cycles_elapsed.avg.per_second','launch__registers_per_thread','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','smsp__inst_executed.sum','lts__t_bytes.sum']
for r in rows[2:]:
    for i,h in enumerate(hdr):
        if h in keys or any(h==k for k in keys): print(f"{h:75s} {units[i]:10s} {r[i]}")
    print('---')
