# Launch list (ncu, one C2 step) of the partitioned gather's kernels next to the one-pass kernel
mkdir -p gpurun_out
Z=${Z:-1.0}
ncu --kernel-name regex:"k_pg|k_gather_vec" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c ${NK:-12} --csv --log-file gpurun_out/pg_ncu_$Z.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu --no-e2e --z $Z > gpurun_out/pg_ncu_$Z.log 2>&1
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/pg_ncu_$Z.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); key=(int(d['ID']),d['Kernel Name'].split('(')[0][-30:])
        data.setdefault(key,{})[d['Metric Name']]=d['Metric Value']
for k,v in sorted(data.items()):
    print(k[0],k[1],'ms=%.3f'%(float(v['gpu__time_duration.sum'])/1e6),'rdGB=%.2f'%(float(v['dram__bytes_read.sum'])/1e9),'wrGB=%.2f'%(float(v['dram__bytes_write.sum'])/1e9),'l2hit=%s'%v.get('lts__t_sector_hit_rate.pct'))
PY
