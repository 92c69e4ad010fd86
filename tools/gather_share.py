"""How many NR factor gathers could rows of a level share? (analysis, host only)

The left-looking block Crout of nr_factor_kernel gathers U^_mt once per
update A_pt -= L^_pm U^_mt of row p. Rows of one elimination level are
independent, so two rows of a level that update from the same source block
(m, t) could gather it once. This counts, on the 2x2-block bus graph in the
plan's ordering, the updates per level and the distinct source blocks among
them: the gather traffic a row-panel (supernodal) schedule could save.

    python tools/gather_share.py [gb2224] [--tail 44]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_14103_b200 import fixtures  # noqa: E402
from paper_2605_14103_b200.transmission import (  # noqa: E402
    build_transmission_model, bus_pattern, jacobian_ordering)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="gb2224")
    ap.add_argument("--tail", type=int, default=44)
    ap.add_argument("--ordering", default="minfill")
    a = ap.parse_args()
    model = build_transmission_model(fixtures.load_transmission(a.case), ordering=a.ordering)
    perm = jacobian_ordering(model)
    pat = bus_pattern(model).tocsr()
    n = pat.shape[0]
    pos = np.empty(n, dtype=np.int64)
    pos[perm] = np.arange(n)
    adj = [set() for _ in range(n)]
    for i in range(n):
        for j in pat.indices[pat.indptr[i]:pat.indptr[i + 1]]:
            if i != j:
                adj[pos[i]].add(int(pos[j]))
    # symbolic elimination in order: higher neighbours of k form a clique
    upper = [None] * n
    for k in range(n):
        hi = sorted(x for x in adj[k] if x > k)
        upper[k] = hi
        for x in hi:
            adj[x].update(y for y in hi if y != x)
    lower = [[] for _ in range(n)]
    for m in range(n):
        for t in upper[m]:
            lower[t].append(m)
    level = np.zeros(n, dtype=np.int64)
    for p in range(n):
        if lower[p]:
            level[p] = 1 + max(level[m] for m in lower[p])
    tail0 = n - a.tail if a.tail > 0 else n
    # updates of row p: source rows m in L(p); targets t in U(m) with t >= p
    # (U part and diagonal) or m < t < p (L part): every t in U(m) that is in
    # row p's pattern, which by fill closure is every t in U(m) with t >= ... ;
    # row p holds columns lower[p] (L) + [p] + upper[p] (U)
    total = 0
    per_level = {}
    for p in range(n):
        rowcols = set(lower[p]) | {p} | set(upper[p])
        lv = int(level[p]) if p < tail0 else -1  # -1: the tail level (non-tail sources only)
        d = per_level.setdefault(lv, [0, set(), 0])
        d[2] += 1
        for m in lower[p]:
            if p >= tail0 and m >= tail0:
                continue  # done densely by nr_tail_kernel
            for t in upper[m]:
                if t in rowcols:
                    total += 1
                    d[0] += 1
                    d[1].add((m, t))
    all_upd = sum(len(upper[m]) and sum(1 for t in upper[m] if t in (set(lower[p]) | {p} | set(upper[p])))
                  for p in range(n) for m in lower[p])
    nnz = n + 2 * sum(len(u) for u in upper)
    print(f"{a.case} ({a.ordering}): {n} block rows, {nnz} blocks, {all_upd} block updates "
          f"(sparse+tail-level {total}, dense tail {all_upd - total}), tail rows {n - tail0}")
    print(f"{'level':>6} {'rows':>5} {'updates':>8} {'distinct':>8} {'share':>6}")
    tot_u = tot_d = 0
    for lv in sorted(per_level, key=lambda x: (x < 0, x)):
        u, s, rows = per_level[lv]
        tot_u += u
        tot_d += len(s)
        name = "tail" if lv < 0 else str(lv)
        if u:
            print(f"{name:>6} {rows:>5} {u:>8} {len(s):>8} {len(s) / u:6.3f}")
    print(f"total updates {tot_u}, distinct per level {tot_d}: a level-shared gather would read "
          f"{tot_d / max(tot_u, 1):.3f} of the update gathers")


if __name__ == "__main__":
    main()
