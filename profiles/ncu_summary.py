"""Text summary of one `ncu --set full --import-source on` capture (one kernel):
    python profiles/ncu_summary.py <file.ncu-rep> [top_n_lines]
Prints selected raw metrics, the stall-reason totals, the hottest SASS lines and the instruction mix."""
import csv,collections,sys,subprocess
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines()))
h=rows[0]; units=rows[1]; r=rows[2]
want=['gpu__time_duration.sum','sm__throughput.avg.pct','smsp__inst_executed.sum','sm__inst_executed_pipe_fma.sum.pct','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct','launch__registers_per_thread','launch__occupancy_limit','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__issue_active.avg.pct','sm__cycles_active.avg','l1tex__data_pipe_lsu_wavefronts.avg.pct','launch__grid_size','smsp__average_warps_issue_stalled','lts__t_bytes.sum ','lts__t_sectors_srcunit_tex_op_read.sum','smsp__cycles_active.avg ','sm__cycles_elapsed.avg ','achieved_occupancy','sm__maximum_warps_per_active_cycle_pct']
for i,name in enumerate(h):
    if any(w in name for w in want) and 'Not Issued' not in name:
        try:
            v=float(r[i].replace(',',''))
            if 'stalled' in name and v<0.05: continue
        except: pass
        print(f"{name:95s} {units[i]:10s} {r[i]}")
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines()))
h=rows[1]; ci={n:i for i,n in enumerate(h)}
data=[]
for rr in rows[2:]:
    if rr and rr[0]=='Kernel Name': break
    if len(rr)>=len(h): data.append(rr)
tot=sum(int(x[ci['# Samples']]) for x in data)
print('total samples',tot,'rows',len(data))
stall_cols=[n for n in h if n.startswith('stall_') and 'Not Issued' not in n]
agg=collections.Counter()
for x in data:
    for c in stall_cols: agg[c]+=int(x[ci[c]])
print({k[6:]:v for k,v in agg.most_common(8)})
top=sorted(data,key=lambda x:-int(x[ci['# Samples']]))[:int(sys.argv[2]) if len(sys.argv)>2 else 14]
for x in top:
    st=sorted(((int(x[ci[c]]),c[6:]) for c in stall_cols),reverse=True)[:2]
    print(f"{int(x[ci['# Samples']]):6d} {100*int(x[ci['# Samples']])/tot:5.1f}% exec={x[ci['Instructions Executed']]:>8s} {x[ci['Source']].strip()[:60]:60s} {st}")
mix=collections.Counter()
for x in data:
    t=x[ci['Source']].strip().split()
    op=t[1] if t[0].startswith('@') else t[0]
    mix[op.split('.')[0]]+=int(x[ci['Instructions Executed']])
ti=sum(mix.values()); print('total inst',ti)
print(' '.join(f"{k}:{100*v/ti:.1f}%" for k,v in mix.most_common(14)))
