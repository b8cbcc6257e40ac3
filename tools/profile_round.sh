# Round profile set: bench line, launch list, ncu --set full of the top kernels.
# usage (on the GPU box): bash tools/profile_round.sh
set -x
B="python bench.py --steps 20 --warmup 3 --no-cpu --e2e-solves 0 --c4-nodes 0 --configs none"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err
timeout 600 $B > gpurun_out/plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_fused_s -s 3 -c 1 -o gpurun_out/prof_kf $B > gpurun_out/ncu_kf.log 2>&1; echo kf_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_prox_window" -s 16 -c 1 -o gpurun_out/prof_k3 $B > gpurun_out/ncu_k3.log 2>&1; echo k3_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kr_reduce" -s 16 -c 1 -o gpurun_out/prof_kr $B > gpurun_out/ncu_kr.log 2>&1; echo kr_rc=$?
timeout 600 $B --engine two_pass > gpurun_out/plain2.log 2>&1; echo plain2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_forward|k2_transpose" -s 30 -c 2 -o gpurun_out/prof_2p $B --engine two_pass > gpurun_out/ncu_2p.log 2>&1; echo 2p_rc=$?
timeout 600 python tools/bench_c4.py 1.0 512 10 > gpurun_out/c4_plain.log 2>&1; echo c4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|kb_window|kb_step|kb_obj|kb_rhs" -s 66 -c 6 -o gpurun_out/prof_tc python tools/bench_c4.py 1.0 512 10 > gpurun_out/ncu_tc.log 2>&1; echo tc_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/bench_c4.py 1.0 512 10 > gpurun_out/c4_ncu.log 2>&1; echo c4l_rc=$?
python tools/ncu_summary.py gpurun_out/ncu_summary.json gpurun_out/prof_kf.ncu-rep gpurun_out/prof_k3.ncu-rep gpurun_out/prof_kr.ncu-rep gpurun_out/prof_2p.ncu-rep gpurun_out/prof_tc.ncu-rep; echo summary_rc=$?
for r in kf k3 kr 2p tc; do ncu -i gpurun_out/prof_$r.ncu-rep --page details --csv > gpurun_out/details_$r.csv 2>/dev/null; done
python tools/ncu_lines.py gpurun_out/prof_kf.ncu-rep kf_fused 60 > gpurun_out/lines_kf.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_tc.ncu-rep tc_gemm 60 > gpurun_out/lines_tc.txt 2>&1
rm -f gpurun_out/prof_k3.ncu-rep gpurun_out/prof_kr.ncu-rep gpurun_out/prof_2p.ncu-rep
du -sh gpurun_out; ls -la gpurun_out
