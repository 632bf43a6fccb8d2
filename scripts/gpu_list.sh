mkdir -p gpurun_out
CMD="python scripts/phase_probe.py ${1:-3} ${2:-bf16}"
$CMD > gpurun_out/plain_list.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none -s 40 -c 20 --csv --log-file gpurun_out/launches_probe.csv $CMD > /dev/null 2>&1
echo "exit $?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_probe.csv')))
for i,r in enumerate(rows):
    if r and r[0]=='ID': hdr=r; start=i+1; break
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
byid={}
for r in rows[start:]:
    if len(r)<=vi: continue
    byid.setdefault(r[ii],{'name':r[ki][:45]})[r[mi]]=r[vi]
for k,v in byid.items(): print(v)
PY
