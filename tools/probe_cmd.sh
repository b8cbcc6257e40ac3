# parity subset, A/B timing, then the per-tile probe timeline (the probe build replaces the .so: run last)
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fista.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
L0_DEBUG=1 timeout 600 python tools/ab_widen.py C5 0.2 50 ${MODES:-1} 2>&1 | grep -v Warn | grep -v "^fused_plan: cs=[1-9][0-9]*.*ncl=0"
timeout 600 python tools/ab_widen.py C3 1.0 100 ${MODES:-1} 2>&1 | grep -v Warn
timeout 600 python tools/ab_widen.py C2 1.0 200 1 2>&1 | grep -v Warn
if [ -n "$PROBE" ]; then
L0_PROBE=1 python -m paper_2502_09502_b200.build --force > gpurun_out/probe_build.log 2>&1
timeout 300 python tools/probe_kfs.py C5 0.2 > gpurun_out/probe_c5.log 2>&1
timeout 300 python tools/probe_kfs.py C3 1.0 > gpurun_out/probe_c3.log 2>&1
head -4 gpurun_out/probe_c5.log gpurun_out/probe_c3.log
fi
