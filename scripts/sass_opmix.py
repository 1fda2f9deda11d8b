"""Static SASS op mix of the hot kernels of libldg_b200.so (cuobjdump -sass):
FP64 / paired-FP32 / FP16 FMAs, vector widths of the global and shared loads.
python scripts/sass_opmix.py [lib] > profiles/rNN_sass_opmix.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1408_3877_b200/libldg_b200.so"
HOT = ["k_s2f<4, 1, uint2, uint2, float>", "k_s2f<3, 1, uint2, uint2, float>", "k_s2f<2, 1, uint2, uint2, float>",
       "k_s1f<4, float, false>", "k_s1f<4, float, true>", "k_s1f<3, float, true>", "k_stage1r<4", "k_stage1m<4",
       "k_stage2<4, true>", "k_stage2<4, false>", "k_full<4, true>",
       "k_assemble_rows<4, 4", "k_assemble_rows<4, 0", "k_bjac_warp<4, 3", "k_dense_gemv", "k_mdot_flat"]
OPS = ["DFMA", "DMUL", "DADD", "FFMA2", "FFMA", "FMUL2", "HFMA2", "HADD2", "F2F", "LDG.E.128", "LDG.E.64",
       "LDG.E.CONSTANT.128", "LDG.E", "LDS.128", "LDS.64", "LDS", "STG.E.128", "STG.E.64", "STG.E", "SHFL",
       "BAR.SYNC", "UTMALDG", "UBLKCP", "HMMA", "DMMA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            for o in OPS:  # longest matching prefix first (OPS ordered so)
                if op == o or op.startswith(o + "."):
                    funcs[cur][o] += 1
                    break
            funcs[cur]["total"] += 1
    names = demangle(list(funcs))
    print(f"# static SASS op mix, {LIB} (cuobjdump -sass; instruction counts in the kernel body, not dynamic)")
    print(f"{'kernel':58s} " + " ".join(f"{o:>9s}" for o in ["total"] + OPS[:8] + ["LDG.E.128", "LDG.E.64", "LDS.128", "STG.E.64"]))
    for hot in HOT:
        for mangled, cnt in funcs.items():
            dn = names[mangled]
            if hot in dn.replace("(anonymous namespace)::", ""):
                short = re.sub(r"\(.*", "", dn.replace("ldgb::(anonymous namespace)::", ""))[:58]
                cols = ["total"] + OPS[:8] + ["LDG.E.128", "LDG.E.64", "LDS.128", "STG.E.64"]
                print(f"{short:58s} " + " ".join(f"{cnt.get(o, 0):9d}" for o in cols))
                break


if __name__ == "__main__":
    main()
