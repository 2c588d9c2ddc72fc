#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the small-size GPU parity
# tests of every family (F: the fused profile + compress pass and its pipelined chain;
# H: the hybrid exchange at W > 1): C1 / edge-layer QSGD (K1 bulk-copy ring, K5, K8, K9, the
# peer-memory exchange on simulated ranks), the DP (16-CTA cluster with DSMEM st.async,
# the two-group join, the one-CTA kernels), TopK, PowerSGD (tcgen05), accumulate.
# Full-size cases are deselected (the tools slow kernels down ~100x).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sanitize
F_Q=tests/test_gpu_qsgd.py
SEL_Q='(test_profile_parity and not adversarial) or test_pack_parity or test_exchange_parity_simulated_ranks or test_compress_allreduce_w1 or test_profile_parity_adversarial_buckets or (test_p2p_exchange_simulated_ranks and 2) or test_golden_packed_record_gpu or (test_accumulate_parity and not 25557032)'
F_D=tests/test_gpu_dp.py
SEL_D='test_random_tables or test_worked_example or (test_narrow_keys_ties_and_bands and (7 or 17)) or test_nonfinite_table or (test_layer_groups_bit_exact and 2)'
F_T=tests/test_gpu_topk.py
SEL_T='test_profile_parity or test_pack_parity or test_exchange_simulated_ranks or test_compress_allreduce_w1_and_nonfinite or test_no_payload_compress_after_payload_compress'
F_P=tests/test_gpu_psgd.py
SEL_P='test_profile_parity or test_profile_exact_low_rank or test_compress_simulated_ranks_two_steps or test_compress_allreduce_w1'
F_F=tests/test_gpu_fused.py
SEL_F='(test_profile_compress_parity and (C1 or edge)) or test_profile_compress_skip_and_bad_choice or (test_pipelined_chain_matches_oracle and C1)'
F_H=tests/test_gpu_hybrid.py
SEL_H='test_hybrid_exchange_simulated_ranks and 2'
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  for fam in ${FAMS:-Q D T P F H}; do
    eval sel=\$SEL_$fam
    eval files=\$F_$fam
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $tool $extra --error-exitcode 7 --print-limit 20 \
      python -m pytest $files -m gpu -q -x -p no:cacheprovider -k "$sel" > gpurun_out/sanitize/${tool}_${fam}.log 2>&1
    echo "$tool $fam exit $?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
