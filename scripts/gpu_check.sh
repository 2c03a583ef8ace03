cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for B in 32 1024; do
echo "B=$B, warm caches (ncu --cache-control none), one in-place step after 10"
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 500 --csv python profiles/warm_l2_step.py $B 2>/dev/null > gpurun_out/warm_$B.csv
python - $B <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f"gpurun_out/warm_{sys.argv[1]}.csv")) if len(r)>5]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value'); i=h.index('ID')
d={}
for r in rows[1:]: d.setdefault(int(r[i]), [r[k], {}])[1][r[m]]=float(r[v].replace(',',''))
ids=sorted(d)
# one step = the launches from the 11th k_frames/first-conv launch: print the last 20 records
for j in ids[-16:]:
    name,x=d[j]; print(f"{name.split('(')[0][:60]:60s} {x.get('gpu__time_duration.sum',0)/1000:7.2f} us  R {x.get('dram__bytes_read.sum',0)/1e6:7.3f} MB  W {x.get('dram__bytes_write.sum',0)/1e6:7.3f} MB")
PY
done
