#!/bin/bash
set -u
mkdir -p gpurun_out/r2q
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
run() {  # name kernel-regex skip
  timeout 900 ncu --set full --clock-control none -k regex:$2 -s $3 -c 1 -o gpurun_out/r2q/$1 python tools/profile_kernels.py $1 > gpurun_out/r2q/$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i gpurun_out/r2q/$1.ncu-rep --page raw --csv > gpurun_out/r2q/$1_raw.csv 2>/dev/null
}
run tf96 hs_jit_eval 2
run ws1000 hs_jit_eval 2
run sa hs_jit_sa 1
run sa_multi hs_jit_sa 1
run ea_multi ea_draw 1
cp gpurun_out/r2q/ea_multi_raw.csv gpurun_out/r2q/ea_draw_raw.csv
timeout 900 ncu --set full --clock-control none -k regex:hs_jit_ea -s 1 -c 1 -o gpurun_out/r2q/ea_chain python tools/profile_kernels.py ea_multi > /dev/null 2>&1; echo "ea chain rc=$?"
ncu -i gpurun_out/r2q/ea_chain.ncu-rep --page raw --csv > gpurun_out/r2q/ea_chain_raw.csv 2>/dev/null
run validate validate 1
rm -f gpurun_out/r2q/*.ncu-rep
ls gpurun_out/r2q
