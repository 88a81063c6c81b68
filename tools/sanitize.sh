# compute-sanitizer memcheck / racecheck / synccheck over the small GPU parity
# cases: BH device build (bottom-up enumeration, bucket pass + climb, edge
# cases), walk + fused force (incl. the overlap queue, the one-kernel overlap
# mode 2 and the staged mode),
# data manager, executor, closed-loop MD, LJ / 2-D MD kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="tests/test_bh_gpu.py::test_fused_ring_edge_cases tests/test_bh_gpu.py::test_golden_tree_lists_forces \
tests/test_bh_gpu.py::test_tiny_softening_finite_and_exact tests/test_bh_gpu.py::test_device_build_edge_cases \
tests/test_bh_gpu.py::test_bucket_tree_reset_equals_fresh_build tests/test_dm_gpu.py tests/test_executor_gpu.py::test_executor_matches_oracle \
tests/test_mdloop_gpu.py::test_device_closed_loop_bit_exact tests/test_md_gpu.py::test_lj_small_vs_oracle_and_bruteforce \
tests/test_md_gpu.py::test_md2d_golden_forces_and_steps"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -p no:cacheprovider -m gpu $T > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
# overlap queue (spin-wait consumer of the walk's published force groups) under memcheck
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -p no:cacheprovider -m gpu \
  tests/test_bh_gpu.py::test_overlapped_step_bit_identical tests/test_bh_gpu.py::test_overlap_theta_change_rewalks \
  > gpurun_out/sanitize_overlap.log 2>&1
echo "overlap memcheck rc=$?" >> gpurun_out/sanitize_overlap.log
