# Round-2 profile set (GPU box): launch list of the C2 bench core, ncu --set
# full of the top kernels per config, summaries for profiles/.
# usage: bash tools/profile_r2.sh
set -x
B="python bench.py --steps 20 --warmup 3 --no-cpu --e2e-solves 0 --c4-nodes 0 --c5-steps 0 --configs none"
timeout 600 $B > gpurun_out/p2_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_launches_c2.csv $B > gpurun_out/p2_ncu_launch.log 2>&1; echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kf_fused_s|k3_prox_window|kr_reduce" -s 30 -c 3 -o gpurun_out/p2_c2 $B > gpurun_out/p2_ncu_c2.log 2>&1; echo c2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_fused_s -s 10 -c 1 -o gpurun_out/p2_c3 python tools/ncu_cfg_kf.py C3 1.0 > gpurun_out/p2_ncu_c3.log 2>&1; echo c3_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_fused_s -s 10 -c 1 -o gpurun_out/p2_c5 python tools/ncu_cfg_kf.py C5 0.2 > gpurun_out/p2_ncu_c5.log 2>&1; echo c5_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|kb_window|kb_step|kb_obj|kb_rhs" -s 160 -c 14 -o gpurun_out/p2_c4 python tools/bench_c4.py 1.0 512 30 > gpurun_out/p2_ncu_c4.log 2>&1; echo c4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mrhs" -s 4 -c 2 -o gpurun_out/p2_bb python tools/bench_bound.py 64 > gpurun_out/p2_ncu_bb.log 2>&1; echo bb_rc=$?
python tools/ncu_summary.py gpurun_out/ncu_summary_r2.json C2=gpurun_out/p2_c2.ncu-rep C3=gpurun_out/p2_c3.ncu-rep C5s=gpurun_out/p2_c5.ncu-rep C4=gpurun_out/p2_c4.ncu-rep C4bound=gpurun_out/p2_bb.ncu-rep; echo summary_rc=$?
for r in c2 c3 c5 c4 bb; do ncu -i gpurun_out/p2_$r.ncu-rep --page details --csv > gpurun_out/p2_details_$r.csv 2>/dev/null; done
python tools/ncu_lines.py gpurun_out/p2_c2.ncu-rep kf_fused 40 > gpurun_out/p2_lines_c2_kf.txt 2>&1
python tools/ncu_lines.py gpurun_out/p2_c5.ncu-rep kf_fused 40 > gpurun_out/p2_lines_c5_kf.txt 2>&1
python tools/ncu_lines.py gpurun_out/p2_c4.ncu-rep tc_gemm 40 > gpurun_out/p2_lines_c4_tc.txt 2>&1
for r in c2 c5; do ncu -i gpurun_out/p2_$r.ncu-rep --page source --csv --print-source cuda,sass > /tmp/p2_src_$r.csv 2>/dev/null; python tools/ncu_stalls.py /tmp/p2_src_$r.csv 30 > gpurun_out/p2_stalls_$r.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep   # the copy-back is capped at 64 MiB: keep the extracted summaries
du -sh gpurun_out
