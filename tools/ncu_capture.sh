# ncu --set full of the four default hot kernels (one launch each, after the same command ran clean
# without ncu), exported to CSV on the box (raw metrics + per-line source stalls).
# usage: TAG=r02a bash tools/ncu_capture.sh   (under gpurun; one GPU)
set -u
T=${TAG:-r02}
O=gpurun_out
mkdir -p $O
cap() {   # name cfg kernel-regex skip [L batch]
  local name=$1 cfg=$2 k=$3 s=$4; shift 4
  if timeout 900 python tools/prof_step.py $cfg "$@" > $O/${T}_${name}_plain.log 2>&1; then
    timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o $O/${T}_${name} python tools/prof_step.py $cfg "$@" > $O/${T}_${name}_ncu.log 2>&1
    ncu -i $O/${T}_${name}.ncu-rep --page raw --csv > $O/${T}_${name}_raw.csv 2>/dev/null
    ncu -i $O/${T}_${name}.ncu-rep --page details --csv > $O/${T}_${name}_details.csv 2>/dev/null
    ncu -i $O/${T}_${name}.ncu-rep --page source --csv --print-source sass > $O/${T}_${name}_source.csv 2>/dev/null
    gzip -f $O/${T}_${name}_source.csv
    rm -f $O/${T}_${name}.ncu-rep
    echo "$name done"
  else
    echo "$name plain run failed"; tail -5 $O/${T}_${name}_plain.log
  fi
}
cap e2_hist E2 bank_hist_kernel 3
cap e2_head E2 bank_head_ws 1
cap e3_pair_tf32 E3 mimo_gemm_pair_tf32 5
cap e4_pair E4 mimo_gemm_pair_kernel 5
