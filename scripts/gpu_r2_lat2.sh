cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin gpurun_out
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench 2>/dev/null || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/lat_launches.csv ./scripts/_bin/latency_bench 500 20 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/lat_launches.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Kernel Name'][:90], d['Grid Size'], d['Block Size'], d['Metric Value'])
PY
