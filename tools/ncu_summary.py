"""Key counters of ncu reports (duration, instructions, IPC, top stalls and pipes):
    python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...]"""
import csv,sys,subprocess
for rep in sys.argv[1:]:
    out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
    r=list(csv.reader(out.splitlines())); h=r[0]
    for v in r[2:]:
        d=dict(zip(h,v))
        print('==',rep, d.get('Kernel Name','')[:60])
        keys=['gpu__time_duration.sum','smsp__inst_executed.sum','sm__inst_executed.avg.per_cycle_active','sm__warps_active.avg.pct_of_peak_sustained_active']
        for k in keys: print(' ',k,d.get(k))
        st=[(k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''),float(x)) for k,x in d.items() if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio') and x]
        st.sort(key=lambda t:-t[1]); print('  stalls',[(a,round(b,2)) for a,b in st[:8]])
        pp=[(k.replace('sm__inst_executed_pipe_','').replace('.avg.pct_of_peak_sustained_active',''),float(x)) for k,x in d.items() if k.startswith('sm__inst_executed_pipe_') and k.endswith('.avg.pct_of_peak_sustained_active') and x]
        pp.sort(key=lambda t:-t[1]); print('  pipes',[(a,round(b,1)) for a,b in pp[:6]])
