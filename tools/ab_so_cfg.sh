# Same-box A/B of prebuilt engine libraries (paper_2502_09502_b200/libl0b200.so.<suffix>)
# on BASELINE configs: bash tools/ab_so_cfg.sh "C2:1.0:200 C5:0.2:50" sfx1 sfx2 ...
CFGS=$1; shift
cd paper_2502_09502_b200; cp libl0b200.so libl0b200.so.orig; cd ..
for rep in 1 2; do
for sfx in "$@"; do
  cp paper_2502_09502_b200/libl0b200.so.$sfx paper_2502_09502_b200/libl0b200.so
  for c in $CFGS; do IFS=: read name sc it <<< "$c"
    timeout 300 python tools/ab_widen.py $name $sc $it 1 2>&1 | grep -v Warn | sed "s/^/$sfx /"
  done
done
done
cp paper_2502_09502_b200/libl0b200.so.orig paper_2502_09502_b200/libl0b200.so
