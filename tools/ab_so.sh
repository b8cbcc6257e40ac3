# A/B of prebuilt engine libraries on C2: bash tools/ab_so.sh suffix1 suffix2 ...
# (each paper_2502_09502_b200/libl0b200.so.<suffix> is swapped in turn; time_drift-style solves)
cd paper_2502_09502_b200
cp libl0b200.so libl0b200.so.orig
for sfx in "$@"; do
  cp "libl0b200.so.$sfx" libl0b200.so
  (cd .. && echo "== $sfx" && timeout 300 python tools/time_drift.py 2>&1 | head -4)
done
cp libl0b200.so.orig libl0b200.so
