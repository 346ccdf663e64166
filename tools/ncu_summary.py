import csv,sys,subprocess
rep=sys.argv[1]; ntiles=float(sys.argv[2])
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines())); h=r[0]; v=r[2]
want=['gpu__time_duration.sum','sm__cycles_elapsed.avg','sm__cycles_elapsed.avg.per_second','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed','sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active','sm__inst_executed_pipe_uniform.sum.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']
for i,k in enumerate(h):
    if k in want: print(f'{k:70s} {v[i]}')
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines())); hh=rows[1]; data=rows[2:]
iS=hh.index('Source'); iE=hh.index('Instructions Executed'); iW=hh.index('Warp Stall Sampling (All Samples)')
from collections import Counter
c=Counter(); s=Counter(); tot=0
for row in data:
    t=row[iS].split()
    if not t: continue
    op=(t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    n=int(row[iE] or 0); c[op]+=n; s[op]+=int(row[iW] or 0); tot+=n
print('inst per tile', tot/ntiles)
print(' '.join(f'{op}:{n/ntiles:.0f}' for op,n in c.most_common(32)))
