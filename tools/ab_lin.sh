# Same-box A/B of the LIN single-pass kernel's plan knobs (rows per tile, cluster size, widening)
run() { env "$@" timeout 300 python tools/ab_widen.py $CFG $SC $IT ${MODES:-3} 2>&1 | grep -v Warn | sed "s/^/$* /"; }
for rep in 1 2; do
CFG=C5 SC=0.2 IT=50
MODES=1,3 run L0_FZ_R=2 L0_FZ_CS=4
MODES=1 run L0_FZ_R=2 L0_FZ_CS=2
MODES=1 run L0_FZ_R=2 L0_FZ_CS=2 L0_FZ_S=3
MODES=1 run L0_FZ_R=2 L0_FZ_CS=2 L0_FZ_SLEEP=200
MODES=1,3 run FP32_FORWARD=1 L0_FZ_R=2 L0_FZ_CS=2
MODES=1 run FP32_FORWARD=1 L0_FZ_R=2 L0_FZ_CS=4
MODES=1 run FP32_FORWARD=1 L0_FZ_R=4 L0_FZ_CS=4
done
