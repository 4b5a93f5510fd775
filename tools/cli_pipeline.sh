#!/usr/bin/env bash
# f2: the CLI's host/device stage overlap (bdsm run, pipelined by default vs --no-pipeline) on a
# generated 200K-vertex / 2M-edge graph with the paper's 50-query sets; stages.csv preprocess ratio.
O=${O:-gpurun_out/cli}
mkdir -p $O
python - <<'PY'
import numpy as np
rng = np.random.default_rng(3)
V, E, L = 200_000, 2_000_000, 8
w = (np.arange(V) + 1.0) ** (-1 / 1.3); w /= w.sum()
u = rng.choice(V, 3 * E, p=w); v = rng.choice(V, 3 * E, p=w)
m = u != v; a = np.minimum(u[m], v[m]); b = np.maximum(u[m], v[m])
k = np.unique(a.astype(np.int64) << 32 | b)[:E]
perm = rng.permutation(V)
with open("/tmp/cli_g.txt", "w") as f:
    lab = rng.integers(0, L, V)
    f.write("".join(f"v {i} {lab[i]}\n" for i in range(V)))
    f.write("".join(f"e {perm[x >> 32]} {perm[x & 0xffffffff]}\n" for x in k.tolist()))
PY
B=paper_2401_17018_b200/bdsm
for mode in pipe nopipe; do
  extra=""; [ $mode = nopipe ] && extra="--no-pipeline"
  t0=$(date +%s.%N)
  $B run --graph /tmp/cli_g.txt --gen-queries sparse,6,50 --gen-stream 0.01,mixed,10 \
     --seed 7 --timeout 600 --out $O/$mode $extra > $O/$mode.out 2> $O/$mode.err
  echo "$mode wall_s $(python -c "print(round($(date +%s.%N) - $t0, 2))")"
  python - $O/$mode <<'PY'
import csv, sys
rows = list(csv.DictReader(open(sys.argv[1] + "/stages.csv")))
pre = sum(float(r["preprocess_s"]) for r in rows); mat = sum(float(r["match_s"]) for r in rows)
print(sys.argv[1], "batches", len(rows), "preprocess_s %.4f match_s %.4f ratio %.3f" % (pre, mat, pre / (pre + mat)))
PY
  cat $O/$mode.out; tail -2 $O/$mode.err
done
cmp $O/pipe/deltas.csv $O/nopipe/deltas.csv && echo "deltas identical"
