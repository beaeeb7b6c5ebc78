#!/bin/bash
# compute-sanitizer passes over a small parity subset (memcheck: out-of-bounds
# and misaligned accesses; racecheck / synccheck: shared-memory hazards and
# barrier misuse in the map, bound, look-back and walk kernels).
mkdir -p gpurun_out
SUB='tests/test_gpu_parity.py -k "known_answer_tests or cfg2_mining or mine_pass1_every_level_vs_reference and popcount or uniform_head_last_width and 0"'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
      -k "test_known_answer_tests and not many or test_cfg2_mining or (test_mine_pass1_every_level_vs_reference and popcount and 0) or (test_uniform_head_last_width_vs_port and 0)" \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
