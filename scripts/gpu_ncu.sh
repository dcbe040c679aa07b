# One `ncu --set full` capture (+ raw / SASS / source pages as CSV) per hot kernel, each after the same
# command has exited 0 without ncu:  gpurun -- 'bash scripts/gpu_ncu.sh'
# Summarise a SASS page with scripts/sass_hotspots.py; copy what should be judged into profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
prof() {  # name op reps cfg kernel-regex skip
  python scripts/prof_op.py $2 $3 $4 > /dev/null && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$5 -s $6 -c 1 -o /tmp/$1 python scripts/prof_op.py $2 $3 $4 > gpurun_out/$1.log 2>&1
  echo "$1 rc $?"
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
prof ncu_c5_hvp1 hvp1 4 C5 stream_kernel 3
prof ncu_c5_hvp8 hvp8 3 C5 stream_dmma 2
prof ncu_c5_third8 third8 3 C5 stream_dmma 2
prof ncu_c4_fgrad fgrad 4 C4 stream_kernel 3
du -sh gpurun_out
