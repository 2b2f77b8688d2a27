#!/bin/bash
# Static look at the persistent kernel's code generation for a set of -D flags (its TU alone, ~1 min):
#   tools/getrf_codegen.sh [-DFOO ...]   -> DMMA loop bodies (instructions, local-memory ops) + spills
out=/tmp/getrf_cg_$$.cubin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cubin -Xptxas -v "$@" -o $out paper_1611_06365_b200/csrc/mla_getrf_prod.cu 2>&1 | grep -A2 "k_getrf\|run_queue" | grep -E "Function|spill|Used"
python tools/sass_loopstat.py $out _Z7k_getrfN3mla9GetrfArgsE | cut -c1-230
rm -f $out
