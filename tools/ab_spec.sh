# Same-box A/B of the SPEC single-pass kernels (non-linear loss, fp32 X) on C3 (no per-kernel events)
run() { env PROFILE=0 "$@" timeout 600 python tools/ab_widen.py C3 1.0 200 ${MODES:-1} 2>&1 | grep -v Warn | sed "s/^/$* /"; }
for rep in 1 2; do
MODES=3 run L0_FZ_SPEC=0
MODES=1 run L0_FZ_SPEC2=0
MODES=1 run L0_FZ_SPEC2=1
MODES=1 run L0_FZ_SPEC2=0 FP32_FORWARD=1
MODES=1 run L0_FZ_SPEC2=1 FP32_FORWARD=1
done
