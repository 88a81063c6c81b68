cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e.log 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_md_gpu.py -k column > gpurun_out/col.log 2>&1
timeout 600 python -c "
import sys, json; sys.path.insert(0,'.')
import bench
class A: steps=3
print(json.dumps(bench.bench_md8m(A())))
" > gpurun_out/md8m_bench.log 2>&1
