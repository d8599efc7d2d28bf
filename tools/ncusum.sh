#!/bin/bash
# Summarise an ncu report: key metrics, stall reasons, top source lines.  tools/ncusum.sh rep [top]
rep=$1; top=${2:-30}
ncu -i $rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
keys=['gpu__time_duration.sum','dram__bytes_read.sum','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','launch__registers_per_thread']
for i,k in enumerate(h):
    if k in keys: print(k, r[1][i], v[i])
st=[(h[i],v[i]) for i in range(len(h)) if 'smsp__average_warps_issue_stalled' in h[i] and h[i].endswith('_per_issue_active.ratio')]
st=sorted(st,key=lambda x:-float(x[1].replace(',','') or 0))[:8]
print(' '.join('%s=%s'%(k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''),x) for k,x in st))
"
ncu -i $rep --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/_src.csv
python profiles/srcprof.py /tmp/_src.csv $top
