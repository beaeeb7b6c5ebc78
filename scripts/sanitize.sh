#!/bin/bash
# compute-sanitizer passes over a parity subset (memcheck: out-of-bounds and
# misaligned accesses; racecheck / synccheck: shared-memory hazards and
# barrier misuse in the map (automaton and chain), bound, look-back and walk
# kernels), plus memcheck over the C++ adaptor test (reference types,
# multi-rank context).
mkdir -p gpurun_out
rm -f gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -q -m gpu -x \
      -k "test_known_answer_tests and not many or test_cfg2_mining or (test_mine_pass1_every_level_vs_reference and popcount and 0) or (test_uniform_head_last_width_vs_port and 0) or (test_chain_uniform_batches_vs_port and 0 and (sparse or dense)) or test_chain_duplicate_episodes or (test_mine_mode_popcount_pass1 and dense)" \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 tests/cpp/_build/adaptor_test \
  > gpurun_out/sanitize_adaptor.txt 2>&1
echo "adaptor memcheck rc=$?" >> gpurun_out/sanitize_summary.txt
