cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin gpurun_out
nvcc -O2 -gencode arch=compute_100a,code=sm_100a scripts/graph_node_cost.cu -o scripts/_bin/graph_node_cost && ./scripts/_bin/graph_node_cost
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench 2>/dev/null
echo "== no graphs"; MVSK_NO_GRAPHS=1 ./scripts/_bin/latency_bench 500 20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 30 --csv --log-file gpurun_out/lat_launches_warm.csv ./scripts/_bin/latency_bench 500 20 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/lat_launches_warm.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Kernel Name'][:60], d['Metric Value'])
PY
