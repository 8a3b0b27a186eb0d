import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if r and r[0]=='ID': hdr=r; start=i; break
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); idi=hdr.index('ID')
d={}
for r in rows[start+1:]:
    if len(r)<len(hdr): continue
    d.setdefault((int(r[idi]), r[ki].split('(')[0][-34:]),{})[r[mi].split('.')[0][:22]]=r[vi]
n=int(sys.argv[2]) if len(sys.argv)>2 else 6
for k in sorted(d)[-n:]: print(k, d[k])
