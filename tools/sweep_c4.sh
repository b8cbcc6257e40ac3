# C4 batched-iteration time under tuning overrides (one process per setting)
for cfg in "" "L0_TC_SFS=1" "L0_TC_SFS=3" "L0_TC_ST=2" "L0_TC_ST=3" "L0_TC_ST=4" "L0_TC_ST=6"; do
  echo "== $cfg: $(env $cfg python tools/ab_sparse_fwd.py --child 1.0 512 100 /tmp/x.npz 2>&1 | tail -1)"
done
L0_DEBUG=1 python tools/bench_c4.py 1.0 512 100 2>&1 | grep -E "tune|profile"
