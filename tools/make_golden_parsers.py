"""Loader golden cases from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_parsers.py

Mutates the case14 MATPOWER text and the IEEE13 feeder document (seeded line
and JSON-tree edits: dropped/duplicated lines, bad tokens, unclosed matrices,
deleted keys, wrong types, unknown buses/phases, scaled admittances and loads,
dropped elements ...), runs the reference's
``parse_matpower_case`` / ``build_ybus`` and ``parse_distribution_json`` /
``build_zbus_model`` on each, and stores the inputs with the reference outcome
(error type and message, or a summary of the parsed model) in
``tests/golden/loader_cases.json.gz``. tests/test_loader_golden.py replays them
against this package on CPU.
"""

from __future__ import annotations

import copy
import gzip
import hashlib
import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import acpflow as ref  # noqa: E402

from paper_2605_14103_b200.fixtures import read_fixture  # noqa: E402

OUT = ROOT / "tests" / "golden" / "loader_cases.json.gz"
N_CASE, N_FEEDER, N_PERTURB = 400, 300, 150


def csr_digest(y) -> str:
    h = hashlib.sha256()
    for a in (y.indptr, y.indices, y.data):
        h.update(a.tobytes())
    return h.hexdigest()


def case_outcome(text: str) -> dict:
    try:
        net = ref.parse_matpower_case(text)
        y = ref.build_ybus(net).complex_csr()
        y.sort_indices()
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"name": net.name, "notes": list(net.notes), "ignored": list(net.ignored_fields),
            "buses": [[b.id, b.kind.value, b.v_set, b.p_gen, b.q_gen] for b in net.buses],
            "n_branches": len(net.branches), "ybus": csr_digest(y)}


def feeder_outcome(text: str) -> dict:
    try:
        net = ref.parse_distribution_json(text)
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "message": str(exc)}
    res = {"buses": [list(b) for b in net.buses], "slack": net.slack_bus,
           "loads": [[ld.kind, ld.bus, ld.phases, ld.s.real, ld.s.imag] for ld in net.loads]}
    try:
        y = ref.build_three_phase_ybus(net)
        y = y.complex_csr() if hasattr(y, "complex_csr") else y
        res["ybus"] = csr_digest(y)
        m = ref.build_zbus_model(net)
        res["v0"] = [[z.real, z.imag] for z in m.v0]
    except Exception as exc:  # noqa: BLE001
        res["model_error"] = type(exc).__name__
        res["model_message"] = str(exc)
    return res


def mutate_case(lines: list, rng: random.Random) -> str:
    out = list(lines)
    for _ in range(rng.randint(1, 3)):
        k = rng.randrange(len(out))
        op = rng.choice(("drop", "dup", "tok", "num", "bracket", "semi"))
        if op == "drop":
            del out[k]
        elif op == "dup":
            out.insert(k, out[k])
        elif op == "tok":
            out[k] = out[k].replace(rng.choice("1203"), rng.choice(["x", "4", "0", "-1", "3", ""]), 1)
        elif op == "num":
            cells = out[k].split("\t")
            if len(cells) > 2:
                cells[rng.randrange(len(cells))] = rng.choice(["0", "-1", "2", "4", "1e-3", "3"])
                out[k] = "\t".join(cells)
        elif op == "bracket":
            out[k] = out[k].replace("]", "", 1) if "]" in out[k] else out[k] + "]"
        else:
            out[k] = out[k].replace(";", ";;", 1)
    return "\n".join(out)


VALUES = [None, 0, 1.5, "", "x", "a", "ab", "ba", "abc", "aa", "d", [], {}, [1, 2], [1, "2"],
          [[1, 0]], "wye", "delta", "650", "632"]


def tree_paths(node, pre=()):
    yield pre
    if isinstance(node, dict):
        for k, v in node.items():
            yield from tree_paths(v, pre + (k,))
    elif isinstance(node, list):
        for k, v in enumerate(node):
            yield from tree_paths(v, pre + (k,))


def mutate_feeder(doc: dict, rng: random.Random) -> str:
    doc = copy.deepcopy(doc)
    for _ in range(rng.randint(1, 2)):
        p = rng.choice([q for q in tree_paths(doc) if q])
        parent = doc
        for k in p[:-1]:
            parent = parent[k]
        u = rng.random()
        if u < 0.3 and isinstance(parent, dict):
            del parent[p[-1]]
        elif u < 0.4 and isinstance(parent, list):
            parent.append(copy.deepcopy(parent[p[-1]]))
        else:
            parent[p[-1]] = copy.deepcopy(rng.choice(VALUES))
    return json.dumps(doc)


def perturb_feeder(doc: dict, rng: random.Random) -> str:
    """Valid-shaped edits: scale numeric leaves, or drop a line/shunt/load element."""
    doc = copy.deepcopy(doc)
    if rng.random() < 0.25:
        section = rng.choice([k for k in ("lines", "shunts", "loads") if doc.get(k)])
        del doc[section][rng.randrange(len(doc[section]))]
        return json.dumps(doc)
    leaves = [q for q in tree_paths(doc) if q and q[0] in ("lines", "shunts", "loads", "slack")]
    for _ in range(rng.randint(1, 4)):
        p = rng.choice(leaves)
        parent = doc
        for k in p[:-1]:
            parent = parent[k]
        if isinstance(parent[p[-1]], float) or (isinstance(parent[p[-1]], int)
                                                 and not isinstance(parent[p[-1]], bool)):
            parent[p[-1]] = parent[p[-1]] * rng.choice([0.0, -1.0, 2.0, 1e-3, 10.0])
    return json.dumps(doc)


def main() -> int:
    rng = random.Random(20260518)
    case_lines = read_fixture("case14.m").splitlines()
    feeder = json.loads(read_fixture("ieee13.json"))
    cases = [{"kind": "matpower", "text": "\n".join(case_lines)}]
    cases += [{"kind": "matpower", "text": mutate_case(case_lines, rng)} for _ in range(N_CASE)]
    cases.append({"kind": "feeder", "text": json.dumps(feeder)})
    cases += [{"kind": "feeder", "text": mutate_feeder(feeder, rng)} for _ in range(N_FEEDER)]
    cases += [{"kind": "feeder", "text": perturb_feeder(feeder, rng)} for _ in range(N_PERTURB)]
    for c in cases:
        c["expect"] = (case_outcome if c["kind"] == "matpower" else feeder_outcome)(c["text"])
    with gzip.open(OUT, "wt") as fh:
        json.dump(cases, fh)
    n_err = sum("error" in c["expect"] for c in cases)
    print(f"{len(cases)} cases ({n_err} rejected by the reference) -> {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
