# The bench's C3 section N times in fresh processes (run-to-run spread, clocks): bash tools/c3_bench_loop.sh [N]
for i in $(seq 1 ${1:-8}); do
  timeout 600 python bench.py --configs C3 --c5-steps 0 --c4-nodes 0 --e2e-solves 0 --no-cpu --steps 20 --warmup 3 2>/dev/null | tail -1 > /tmp/c3line.json
  python - <<'PY'
import json
c = json.load(open("/tmp/c3line.json"))["other_configs"][0]
print(round(c["value"], 1), round(c["ms_per_iteration"] * c["iterations"], 1), round(c["host_wall_ms"], 1),
      c["gpu_launches"], c["prox_full_passes"], c["restarts"], c["clocks"])
PY
done
