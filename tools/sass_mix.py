"""Static SASS instruction mix of the hot kernels in libacpf.so (cuobjdump -sass).

    python tools/sass_mix.py [paper_2605_14103_b200/libacpf.so] > profiles/r2/sass_mix.txt

For each kernel: instruction count and the mnemonics that show which
Blackwell paths it uses: DMMA (FP64 tensor pipe, mma.sync.m8n8k4.f64),
UBLKCP (cp.async.bulk / TMA bulk engine), LDGSTS (cp.async), SYNCS (mbarrier),
DFMA/DMUL/DADD (FP64 pipe), LDS/STS (shared), LDG/STG (global), SHFL.
"""
import collections
import re
import subprocess
import sys

KEYS = ["DMMA", "UBLKCP", "UTMALDG", "UTCHMMA", "LDGSTS", "SYNCS", "DFMA", "DMUL", "DADD", "MUFU",
        "LDS", "STS", "LDG", "STG", "SHFL", "BAR", "ATOMG", "RED"]
HOT = ["zbus_kernel", "nr_factor_kernel", "nr_back_kernel", "nr_mismatch_kernel", "nr_jacobian_kernel",
       "nr_shared_step_kernel", "nr_phasor_kernel", "nr_tail_kernel", "nr_cond_kernel", "nr_scenarios",
       "zb_scenarios", "nr_cert", "zb_kcl", "fd_gemm_kernel"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_14103_b200/libacpf.so"
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    print(f"# cuobjdump -sass {lib}: static instruction mix of the hot kernels (sm_100a)")
    for f in re.split(r"\n\s*Function : ", txt)[1:]:
        name = f.split("\n", 1)[0].strip()
        short = next((h for h in HOT if h in name), None)
        if not short:
            continue
        ops = collections.Counter()
        for line in f.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(1)] += 1
        tmpl = re.search(r"PipeLdgstsILi(\d)ELi(\d+)ELi(\d+)", name)
        label = short + (f"<NG={tmpl.group(1)},CH={tmpl.group(2)},NBUF={tmpl.group(3)}>" if tmpl else
                         ("<64>" if "ILi64E" in name else "<32>" if "ILi32E" in name else ""))
        tot = sum(ops.values())
        print(f"{label:44s} instr {tot:6d}  " + " ".join(f"{k}:{ops[k]}" for k in KEYS if ops[k]))


if __name__ == "__main__":
    main()
