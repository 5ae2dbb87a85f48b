REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2k_c3_launches.csv python tools/ab_layout.py 512,16384,512 2048,16384,64 > gpurun_out/r2k_c3.log 2>&1
REPS=3 timeout 600 ncu --set full --clock-control none -k regex:stats1 --launch-skip 2 --launch-count 1 -o gpurun_out/r2k_stats1 -f python tools/ab_layout.py 512,16384,512 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r2k_c3_launches.csv')) if len(r)>10 and r[0].isdigit()]
hdr=None
for r in csv.reader(open('gpurun_out/r2k_c3_launches.csv')):
    if r and r[0]=='ID': hdr=r; break
iname=hdr.index('Kernel Name'); imet=hdr.index('Metric Name'); ival=hdr.index('Metric Value'); iid=hdr.index('ID')
out={}
for r in rows:
    out.setdefault(r[iid],{'name':r[iname][:60]})[r[imet]]=r[ival]
for k,v in list(out.items())[-40:]:
    print(k, v['name'], v.get('gpu__time_duration.sum'), v.get('dram__bytes_read.sum'), v.get('dram__bytes_write.sum'))
PY
