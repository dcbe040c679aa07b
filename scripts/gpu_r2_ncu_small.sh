cd $GRAFT_REPO_ROOT
mkdir -p scripts/_bin gpurun_out
nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build -o scripts/_bin/latency_bench 2>/dev/null
name=r2_small_fgrad
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:stream_kernel -s 25 -c 1 -o /tmp/$name ./scripts/_bin/latency_bench 500 20 > gpurun_out/$name.log 2>&1
echo "ncu rc $?"
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
