# ncu --set full of the fp32 single-pass kernel on C3 (full) and C5 (n = 200k rows)
# usage (GPU box): bash tools/prof_kf32.sh [tag]
T=${1:-kf32}
timeout 600 python tools/ncu_cfg_kf.py C3 1.0 > gpurun_out/${T}_c3_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_fused_s -s 10 -c 1 -o gpurun_out/${T}_c3 python tools/ncu_cfg_kf.py C3 1.0 > gpurun_out/${T}_c3_ncu.log 2>&1; echo c3_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_fused_s -s 10 -c 1 -o gpurun_out/${T}_c5 python tools/ncu_cfg_kf.py C5 0.2 > gpurun_out/${T}_c5_ncu.log 2>&1; echo c5_rc=$?
for r in c3 c5; do
  ncu -i gpurun_out/${T}_$r.ncu-rep --page details --csv > gpurun_out/${T}_${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/${T}_$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_${r}_source.csv 2>/dev/null
  ncu -i gpurun_out/${T}_$r.ncu-rep --page raw --csv > gpurun_out/${T}_${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out | tail -20
