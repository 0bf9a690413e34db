# Launch list (ncu, --clock-control none) of the partitioned gather's kernels on the C2 column
# at skew $Z, reordered layout, path forced on (policy 8321 | 16384)
mkdir -p gpurun_out
Z=${Z:-0.5}
ncu --kernel-name regex:"k_pg|k_gather_vec" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c ${NK:-40} --csv --log-file gpurun_out/pg_forced_$Z.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu --no-e2e --z $Z --policy 24705 > gpurun_out/pg_forced_$Z.log 2>&1
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/pg_forced_$Z.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); key=(int(d['ID']),d['Kernel Name'].split('(')[0][-30:])
        data.setdefault(key,{})[d['Metric Name']]=d['Metric Value']
for k,v in sorted(data.items())[-8:]:
    f=lambda m: float(v[m].replace(',',''))
    print(k[0],k[1],'ms=%.3f'%(f('gpu__time_duration.sum')/1e6),'rdGB=%.2f'%(f('dram__bytes_read.sum')/1e9),'wrGB=%.2f'%(f('dram__bytes_write.sum')/1e9),'l2hit=%s'%v.get('lts__t_sector_hit_rate.pct'),'inst=%.2fG'%(f('sm__inst_executed.sum')/1e9),'issue=%s'%v.get('smsp__issue_active.avg.pct_of_peak_sustained_active'))
PY
