"""Executed SASS opcode mix from an ncu --page source --csv --print-source sass export: sass_exec_mix.py src.csv [norm] [top]."""
import csv,sys,collections,re
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; iS=h.index('Source'); iE=h.index('Instructions Executed')
c=collections.Counter(); tot=0
for r in rows[2:]:
    if len(r)<=iE: continue
    try: n=int(r[iE])
    except: continue
    src=r[iS].strip()
    m=re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_.]+)',src)
    op=m.group(2) if m else src
    c[op]+=n; tot+=n
norm=float(sys.argv[2]) if len(sys.argv)>2 else 1
print('total',tot, tot/norm)
for k,v in c.most_common(int(sys.argv[3]) if len(sys.argv)>3 else 30): print(f"{k:28s} {v/norm:10.2f} {100*v/tot:5.1f}%")
