cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc $?"; tail -6 gpurun_out/r2l_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
