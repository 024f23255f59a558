#!/bin/bash
# compute-sanitizer memcheck + racecheck over the GPU parity/codec tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
# (the single-read pack and the fed decode spin on co-resident CTAs, which the
# sanitizer serialises: they are left out)
SEL='(test_restore_paged_matches_oracle or test_fused_pack_matches_oracle or test_golden_streams_decode or test_random_sequences_batched or test_encode_bit_exact or test_restore_batch_mixed or test_pack_paged_source or test_part_pipeline_many_parts or test_tiny_and_ragged or test_large_r1080 or test_all_tilings or supplied_maxima or head_window) and not single_read'
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_codec.py -q -x -k "$SEL" \
      > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.txt | tail -3
done
