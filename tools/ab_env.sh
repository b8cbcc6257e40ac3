# Same-box A/B of an environment knob on BASELINE configs:
# bash tools/ab_env.sh VAR "v1 v2 ..." "C2:1.0:200 C5:0.2:50"
VAR=$1; VALS=$2; CFGS=$3
for rep in 1 2; do
for v in $VALS; do
  for c in $CFGS; do IFS=: read name sc it <<< "$c"
    env $VAR=$v timeout 300 python tools/ab_widen.py $name $sc $it 1 2>&1 | grep -v Warn | sed "s/^/$VAR=$v /"
  done
done
done
