"""Per-opcode stall reasons of an ncu source page (SASS CSV): usage ncu_stall_ops.py src.csv"""
import csv,sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; ix={h:i for i,h in enumerate(hdr)}
cols=['stall_dispatch','stall_short_sb','stall_long_sb','stall_barrier','stall_wait','stall_not_selected','stall_selected','stall_math','stall_mio','stall_branch_resolving','stall_no_inst','stall_lg']
agg=defaultdict(lambda: defaultdict(float))
top=[]
for r in rows[2:]:
    if r and r[0]=="Kernel Name": break
    if len(r)<len(hdr): continue
    src=r[ix['Source']].strip(); op=src.split()[0] if src else '?'
    if op.startswith('@'): op=src.split()[1]
    op=op.split('.')[0]
    for c in cols:
        v=float(r[ix[c]] or 0); agg[op][c]+=v
    top.append((float(r[ix['stall_dispatch']] or 0), r[ix['Address']] if 'Address' in ix else '', src))
tot={c:sum(agg[o][c] for o in agg) for c in cols}
print({c:int(v) for c,v in tot.items()})
for c in ['stall_dispatch','stall_short_sb','stall_long_sb','stall_barrier','stall_wait','stall_branch_resolving','stall_no_inst']:
    items=sorted(((agg[o][c],o) for o in agg), reverse=True)[:5]
    print(c, [(o,int(v)) for v,o in items])
top.sort(reverse=True)
for t in top[:12]: print(t)
