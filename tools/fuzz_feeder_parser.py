"""Differential fuzz: reference parse_distribution_json / build_zbus_model vs ours
on mutated ieee13 documents (build container only; reads /root/reference)."""
import copy
import json
import random
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import acpflow as ref  # noqa: E402
import numpy as np  # noqa: E402

import paper_2605_14103_b200 as me  # noqa: E402
from paper_2605_14103_b200.fixtures import read_fixture  # noqa: E402

BASE = json.loads(read_fixture("ieee13.json"))
VALUES = [None, 0, 1.5, "", "x", "a", "ab", "ba", "abc", "aa", "d", [], {}, [1, 2], [1, "2"],
          [[1, 0]], "wye", "delta", "650", "632"]


def paths(node, pre=()):
    yield pre
    if isinstance(node, dict):
        for k, v in node.items():
            yield from paths(v, pre + (k,))
    elif isinstance(node, list):
        for k, v in enumerate(node):
            yield from paths(v, pre + (k,))


def mutate(doc, rng):
    ps = [p for p in paths(doc) if p]
    p = rng.choice(ps)
    parent = doc
    for k in p[:-1]:
        parent = parent[k]
    op = rng.random()
    if op < 0.3 and isinstance(parent, dict):
        del parent[p[-1]]
    elif op < 0.4 and isinstance(parent, list):
        parent.append(copy.deepcopy(parent[p[-1]]))
    else:
        parent[p[-1]] = copy.deepcopy(rng.choice(VALUES))


def outcome(mod, text):
    try:
        net = mod.parse_distribution_json(text)
    except Exception as e:  # noqa: BLE001
        return ("parse-err", type(e).__name__, str(e))
    try:
        m = mod.build_zbus_model(net)
        return ("ok", net.buses, net.slack_bus, tuple((l.kind, l.bus, l.phases, l.s) for l in net.loads), m.v0.tobytes(),
                m.wye_idx.tobytes(), m.delta_p.tobytes(), m.delta_q.tobytes(),
                me.build_three_phase_ybus(net).data.tobytes() if mod is me else ref.build_three_phase_ybus(net).complex_csr().data.tobytes() if hasattr(ref.build_three_phase_ybus(net), "complex_csr") else ref.build_three_phase_ybus(net).data.tobytes())
    except Exception as e:  # noqa: BLE001
        return ("model-err", type(e).__name__, str(e))


def main(n=1500, seed=3):
    rng = random.Random(seed)
    bad = 0
    for _ in range(n):
        doc = copy.deepcopy(BASE)
        for _ in range(rng.randint(1, 2)):
            mutate(doc, rng)
        text = json.dumps(doc)
        a, b = outcome(ref, text), outcome(me, text)
        if a[0] != b[0] or a[1:3] != b[1:3] or (a[0] == "ok" and a != b):
            bad += 1
            if bad <= 5:
                print("MISMATCH\n ref:", str(a)[:300], "\n  me:", str(b)[:300])
    print("cases", n, "mismatches", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
