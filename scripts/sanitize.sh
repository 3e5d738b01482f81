#!/usr/bin/env bash
# compute-sanitizer passes over small solves of every kernel family (run on the GPU box).
# Usage: gpurun -- bash scripts/sanitize.sh [tag]
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
cat > /tmp/san_run.py <<'EOF'
import sys
sys.path.insert(0, ".")
import chaingen as G
import paper_1911_13214_b200 as R
import os
rng = G.SplitMix64(3)
# L = 230 (8 tile blocks: middle launches up to delta = 7, every leaf / product
# phase), S = 520 (17 m-chunks of the middle, 5 leaf chunks), both schedules
for L, S in [(230, 520), (70, 45), (33, 20)]:
    ch = G.random_chain(rng, L, real_times=True, big=True)
    M = int(sum(int(x) for x in ch.wbx) * 0.25)
    for k, sch in (("tiled", "dag"), ("tiled", "diagonal"), ("wavefront", "dag")):
        if L > 100 and k == "wavefront" and os.environ.get("SAN_FAST"):
            continue
        r = R.solve(ch, M, S, kernel=k, schedule=sch)
        print(k, sch, L, S, r.status, r.cost, r.n_ops)
    R.export_tables(L + 1, S)
r = R.solve_sharded(ch, M, S, [0, 0], halo_mode=1)
print("sharded", r.status, r.cost)
chains, limits, S = G.config5(n_limits=3)
costs, status, n_ops, ops = R.solve_batch(chains[:3], [l[:3] for l in limits[:3]], 60, with_ops=True)
print("batch", costs.shape, status.tolist())
EOF
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 200 python /tmp/san_run.py > "$OUT/$tool.log" 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$OUT/$tool.log" | tail -1)"
done
