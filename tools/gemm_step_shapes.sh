#!/bin/bash
# vp_gemm_bf16 vs cuBLAS at the GPT-2 355M m=32 step shapes (T = 32768 tokens),
# each with the epilogue the executor uses: python tools/microbench.py one M N K layout epi
# epi: 0 STORE 1 BIAS 2 BIAS_GELU 3 BIAS_RESID 4 DGELU 5 ACC_F32
for spec in "32768 3072 1024 nt 1" "32768 1024 1024 nt 3" "32768 4096 1024 nt 2" "32768 1024 4096 nt 3" \
            "32768 4096 1024 nn 4" "32768 1024 4096 nn 0" "32768 3072 1024 nn 0" "32768 1024 1024 nn 0" \
            "4096 1024 32768 tn 5" "1024 4096 32768 tn 5" "3072 1024 32768 tn 5" "1024 1024 32768 tn 5" \
            "32768 4096 1024 nt 0" "32768 51200 1024 nt 0"; do
  timeout 120 python tools/microbench.py one $spec
done
