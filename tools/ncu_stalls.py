"""Per-kernel key metrics and the top warp-stall reasons of an ncu report (read with ncu -i).
  python tools/ncu_stalls.py report.ncu-rep"""
import csv, sys, subprocess, io
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
hdr=rows[0]
keys=['gpu__time_duration.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','lts__t_bytes.sum','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__t_bytes.sum','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:40], r[hdr.index('launch__grid_size')] if 'launch__grid_size' in hdr else '')
    for k in keys:
        if k in hdr: print('   %-70s %s %s'%(k, r[hdr.index(k)], rows[1][hdr.index(k)]))
    st=[]
    for h,v in zip(hdr,r):
        if 'issue_stalled' in h and h.endswith('per_issue_active.ratio'):
            try: st.append((float(v.replace(',','')), h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')))
            except: pass
    print('   stalls:', ', '.join('%s %.2f'%(n,v) for v,n in sorted(st,reverse=True)[:7]))
