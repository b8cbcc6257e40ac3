# Same-box A/B of the fp64 LIN plan: 1-row x 4096-column tiles in clusters of 4 (L0_FZ_WIDE=1) vs 2 x 2048 in clusters of 8
run() { env "$@" timeout 600 python tools/ab_widen.py C2 1.0 200 1 2>&1 | grep -v Warn | sed "s/^/$* /"; }
for rep in 1 2 3; do
run L0_FZ_WIDE=0
run L0_FZ_WIDE=1
run L0_FZ_WIDE=1 L0_FZ_SLEEP=200
done
