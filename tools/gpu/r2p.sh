# memcheck (one sanitizer tool) over a representative set of small GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_batch.py tests/test_shard.py -m gpu -x -q -p no:cacheprovider \
  -k "c1_blob_grid_all_groups or adversarial_masks or wide_grey_levels or large_roi or banded_host_path_bitwise or multi_batch_matches_single or multi_slide_matches_single or batch_mixed" \
  > $O/r2p_memcheck.log 2>&1; echo "rc=$?" >> $O/r2p_memcheck.log
tail -15 $O/r2p_memcheck.log
