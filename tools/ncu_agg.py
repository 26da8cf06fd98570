import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
hdr=rows[0]; data=rows[1:]
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ui=hdr.index('Metric Unit')
agg=collections.OrderedDict()
SC={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
for r in data:
    k=r[ki][:40]; m=r[mi]; v=float(r[vi].replace(',','')); u=r[ui]
    e=agg.setdefault(k,collections.defaultdict(float))
    if m=='gpu__time_duration.sum': e['n']+=1; e['ms']+= v/1e6 if u=='ns' else (v/1e3 if u=='us' else v)
    else: e[m]+=v*SC.get(u,1)
for k,e in agg.items():
    n=e['n']
    print(f"{k:40s} n={n:3.0f} {e['ms']/n:8.3f} ms  dram rd {e['dram__bytes_read.sum']/n/1e9:6.2f} GB wr {e['dram__bytes_write.sum']/n/1e9:6.2f} GB  smem wf {e['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']/n/1e6:8.1f}M conflicts {e['l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']/n/1e6:8.1f}M")
