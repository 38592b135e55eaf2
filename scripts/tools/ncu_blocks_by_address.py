"""Straight-line blocks of an ncu SASS source page in address order, with each
block's share of the executed warp instructions, stall samples, average
active threads and instruction mix -- the view the round-2 instruction
trimming and the packed variance fits came from.

  ncu -i rep.ncu-rep --page source --csv --print-source sass > PREFIX_sass.csv
  ncu -i rep.ncu-rep --page raw --csv > PREFIX_raw.csv
  python scripts/tools/ncu_blocks_by_address.py PREFIX [min share %]
"""
import csv,sys,collections
pre=sys.argv[1]
rows=list(csv.reader(open(pre+'_raw.csv')))
h=rows[0]; v=rows[2]
want=['gpu__time_duration.sum','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__block_size','launch__shared_mem_per_block_static']
for k in want:
    for i,n in enumerate(h):
        if n==k: print(k, v[i])
rows=list(csv.reader(open(pre+'_sass.csv')))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
data=rows[2:]
def f(r,k):
    try: return float(r[idx[k]].replace(',',''))
    except: return 0.0
tot=sum(f(r,"Instructions Executed") for r in data)
tots=sum(f(r,"Warp Stall Sampling (All Samples)") for r in data)
blocks=[];cur=None
for i,r in enumerate(data):
    ex=f(r,"Instructions Executed")
    src=r[idx['Source']]
    op=(src.split()[1] if src.startswith('@') else src.split()[0]) if src.split() else '?'
    if cur and abs(ex-cur['exec'])<1e-6:
        cur['n']+=1; cur['samp']+=f(r,"Warp Stall Sampling (All Samples)"); cur['ops'][op.split('.')[0]]+=1
    else:
        if cur: blocks.append(cur)
        cur={'start':i,'exec':ex,'n':1,'samp':f(r,"Warp Stall Sampling (All Samples)"),'ops':collections.Counter({op.split('.')[0]:1}),'thr':f(r,"Avg. Threads Executed")}
blocks.append(cur)
print('total inst',tot,'lines',len(data))
thr=float(sys.argv[2]) if len(sys.argv)>2 else 1.0
for b in blocks:
    sh=100*b['exec']*b['n']/tot
    if sh>=thr:
        print(f"@{b['start']:5d} n={b['n']:4d} exec={b['exec']:9.0f} inst={sh:5.1f}% samp={100*b['samp']/tots:5.1f}% thr={b['thr']:.0f} {dict(b['ops'].most_common(8))}")
