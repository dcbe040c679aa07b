# A/B of the default build against paper_2604_25378_b200/_build_ab (an alternative build of the library):
#   bash scripts/gpu_r2_ab.sh <out-name> <cfg> <ops> [more "cfg ops" pairs...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/$1.txt; shift
AB=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build_ab/libmvsk_b200.so
{
for rep in 1 2; do
  set -- "$@"
  args=("$@")
  for ((i=0; i<${#args[@]}; i+=2)); do
    echo "== new ${args[i]}"; timeout 300 python scripts/dmma_ab.py ${args[i]} ${args[i+1]} ws
    echo "== base ${args[i]}"; MVSK_B200_LIB=$AB timeout 300 python scripts/dmma_ab.py ${args[i]} ${args[i+1]} ws
  done
done
} > $out 2>&1
cat $out
