# Same-box A/B of programmatic dependent launch on the single-pass chain (L0_PDL)
run() { env PROFILE=0 "$@" timeout 300 python tools/ab_widen.py $CFG $SC $IT 1 2>&1 | grep -v Warn | sed "s/^/$* /"; }
for rep in 1 2; do
for v in 0 1; do
CFG=C2 SC=1.0 IT=200 run L0_PDL=$v
CFG=C3 SC=1.0 IT=200 run L0_PDL=$v
CFG=C5 SC=0.2 IT=50 run L0_PDL=$v
done
done
