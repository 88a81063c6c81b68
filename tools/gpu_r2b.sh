cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_bh_gpu.py -k "oracle_tree" > gpurun_out/tree.log 2>&1; echo "rc=$?" >> gpurun_out/tree.log
bash tools/sanitize.sh
