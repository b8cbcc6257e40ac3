# ncu --set full of the fp32 single-pass kernel on C5 (n = 200k rows) [and C3 full]
# usage (GPU box): bash tools/prof_kf32.sh [tag] [configs...]
T=${1:-kf32}; shift
CFGS=${@:-c5}
for c in $CFGS; do
  case $c in c3) A="C3 1.0";; c5) A="C5 0.2";; c2) A="C2 1.0";; esac
  timeout 600 python tools/ncu_cfg_kf.py $A > gpurun_out/${T}_${c}_plain.log 2>&1; echo ${c}_plain_rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_fused_s -s 10 -c 1 -o gpurun_out/${T}_$c python tools/ncu_cfg_kf.py $A > gpurun_out/${T}_${c}_ncu.log 2>&1; echo ${c}_rc=$?
  ncu -i gpurun_out/${T}_$c.ncu-rep --page details --csv > gpurun_out/${T}_${c}_details.csv 2>/dev/null
  ncu -i gpurun_out/${T}_$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_${c}_source.csv 2>/dev/null
  ncu -i gpurun_out/${T}_$c.ncu-rep --page raw --csv > gpurun_out/${T}_${c}_raw.csv 2>/dev/null
done
ls -la gpurun_out | tail -12
