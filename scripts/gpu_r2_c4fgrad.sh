cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/tune_vs.py C4 2>&1 | grep "default"
prof() {  # name kernel-regex skip cmd...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --warp-sampling-interval 0 --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
  echo "$name rc $?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
  rm -f /tmp/$name.ncu-rep
}
prof r2_c4_fgrad_rg2 stream_kernel 3 python scripts/prof_op.py fgrad 4 C4
prof r2_gpcg_cluster2 gram_pcg_cluster 5 python scripts/one_solve_prof.py C4
