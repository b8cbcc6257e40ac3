# KF variants on C2: bench line per setting (usage: bash tools/sweep_kf.sh "ENV=.. ENV=.." ...)
B="python bench.py --steps 100 --warmup 3 --no-cpu --e2e-solves 0 --c4-nodes 0 --configs none --engine single_pass"
for cfg in "$@"; do
  echo "== $cfg"; env $cfg L0_DEBUG=1 timeout 300 $B 2>&1 | grep -E "fused_plan|\[bench\] 100|rror" | tail -4
done
