#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (one or two small
# solves each; summaries to gpurun_out/sanitize_<tool>.txt)
cd "$(dirname "$0")/.."
python -c "import paper_0907_4631_b200 as P; P.build()"
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=(
  "c1_mini|--expm 0|single-CTA Krylov + DMMA Taylor expm"
  "c1_mini|--expm 1|Pade-13 expm"
  "c1_mini|--expm 2|Chebyshev phi kernel"
  "c2_med||persistent Lanczos (smem) + cooperative w-recurrence"
  "c3_med|--option persist=0|streaming TMA-halo SpMV + axpy (two-kernel Arnoldi, lagged)"
  "c3_med||persistent Arnoldi"
  "c4_tm|--option brick=0|TMEM persistent Lanczos + cooperative w-recurrence"
  "c4_tm|--option brick=2|brick Lanczos + brick w-recurrence (tensor-map TMA, TMEM; ragged x segments)"
  "c5_med||CSR ELL x-ring SpMV + CSR analysis"
)
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/sanitize_$tool.txt; : > $out
  for c in "${CASES[@]}"; do
    IFS='|' read -r cfg opts what <<< "$c"
    echo "=== $tool: $cfg $opts ($what)" >> $out
    timeout 600 $CS --tool $tool --print-limit 20 python tools/one_solve.py --config $cfg --solves 1 $opts > /tmp/san.log 2>&1
    echo "exit=$?" >> $out
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|hazard|Barrier|error" /tmp/san.log | head -20 >> $out
    tail -2 /tmp/san.log >> $out
  done
done
cat gpurun_out/sanitize_*.txt
