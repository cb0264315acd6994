#!/bin/bash
# which earlier test on the session context breaks the c2 trajectory test
T=tests/test_gpu_solve.py
TGT="$T::test_controller_trajectory_matches_oracle[c2-stencil]"
for k in test_solve_parity_small test_solve_parity_pade13 test_solve_parity_full_configs test_csr_and_stencil_agree test_all_p test_multistep_stiff test_cgs2_and_fixed_m test_fixed_m_phip_parity test_eq6_variant test_degenerate_inputs test_a_zero_and_tiny_n test_host_buffers_match_device test_deterministic test_profile_counts test_stencil_arnoldi_early_breakdown; do
  r=$(timeout 300 python -m pytest -q -p no:cacheprovider "$T::$k" "$TGT" 2>&1 | tail -1)
  echo "$k: $r"
done
