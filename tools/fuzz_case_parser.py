"""Differential fuzz: reference parse_matpower_case vs ours on mutated case14 text (build container only)."""
import sys, random, re
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import acpflow as ref
import paper_2605_14103_b200 as me
from paper_2605_14103_b200.fixtures import read_fixture
base = read_fixture("case14.m")
lines = base.splitlines()
rng = random.Random(1)
def res(mod, text):
    try:
        n = mod.parse_matpower_case(text)
        return ("ok", n.name, [(b.id, b.kind.value, b.v_set, b.p_gen, b.theta_set) for b in n.buses],
                [tuple(vars(b).values()) for b in n.branches], n.notes, n.ignored_fields)
    except Exception as e:
        return ("err", type(e).__name__, str(e))
mism = 0
muts = ["drop", "dup", "tok", "num", "bracket", "semi"]
for it in range(3000):
    L = list(lines)
    for _ in range(rng.randint(1, 3)):
        k = rng.randrange(len(L)); m = rng.choice(muts)
        if m == "drop": del L[k]
        elif m == "dup": L.insert(k, L[k])
        elif m == "tok": L[k] = L[k].replace(rng.choice(["1", "2", "0", "3"]), rng.choice(["x", "4", "0", "-1", "3", ""]), 1)
        elif m == "num":
            toks = L[k].split("\t")
            if len(toks) > 2:
                j = rng.randrange(len(toks)); toks[j] = rng.choice(["0", "-1", "2", "4", "1e-3", "3"]); L[k] = "\t".join(toks)
        elif m == "bracket": L[k] = L[k].replace("]", "", 1) if "]" in L[k] else L[k] + "]"
        elif m == "semi": L[k] = L[k].replace(";", ";;", 1)
    t = "\n".join(L)
    a, b = res(ref, t), res(me, t)
    if a[0] != b[0] or (a[0] == "err" and a[2] != b[2]) or (a[0] == "ok" and a != b):
        mism += 1
        if mism < 5: print("MISMATCH", a[:3] if a[0]=="err" else a[0], "|", b[:3] if b[0]=="err" else b[0])
print("mismatches", mism)
