"""SASS evidence for the hot kernels of the built library (cuobjdump -sass):
per kernel the mnemonic counts that prove the pipe (UTCHMMA / UTMALDG / LDTM
for tcgen05 + TMA, DMMA, DFMA, HADD2 / HFMA2 / HMUL2 for f16x2) and an
excerpt of the innermost loop (the longest straight run between a backward
branch's target and the branch). Usage: python tools/sass_excerpts.py [lib]"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2311_15393_b200/_lib/libkronprec_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
WANT = [("gemm_f16x_kernel", "gemm_f16x (tcgen05 rounded leaves + HADD2 trees)"),
        ("gemm_f16ref_kernelILi2ELi64ELi64", "gemm_f16ref <2,64,BN=64> (HMUL2 + HADD2)"),
        ("gemm_f16tc_kernelILi256", "gemm_f16tc <BN=256> (tensor mode, tcgen05 fp32 accumulate)"),
        ("gemm_f64_kernelILi64ELi64ELi32ELi32ELi4ELi1ELb0", "gemm_f64 (DMMA operator GEMM)"),
        ("band_cols_kernelILi41", "band_cols<41> (banded pass A, DFMA)"),
        ("band_rows_kernelILi41", "band_rows<41> (banded pass B, DFMA)")]
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "LDTM", "DMMA", "DFMA", "DADD", "DMUL", "HADD2", "HFMA2", "HMUL2",
        "LDS", "LDSM", "LDGSTS", "STS", "SYNCS", "BAR"]
for key, title in WANT:
    body = next((f for f in funcs if f.split("\n", 1)[0].find(key) >= 0), None)
    if body is None:
        print(f"== {title}: not found")
        continue
    lines = [ln for ln in body.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", ln)]
    ops = collections.Counter()
    for ln in lines:
        m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            ops[m.group(2)] += 1
    print(f"== {title}  ({body.split(chr(10), 1)[0].strip()[:90]})")
    print("   " + "  ".join(f"{k}:{ops[k]}" for k in KEYS if ops[k]))
    # innermost loop: backward BRA with the shortest span containing the most hot ops
    addr = {}
    for idx, ln in enumerate(lines):
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m:
            addr[int(m.group(1), 16)] = idx
    best = None
    for idx, ln in enumerate(lines):
        m = re.search(r"BRA\s+(?:`\()?\.?L?_?x?_?(0x[0-9a-f]+)", ln)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt in addr and addr[tgt] < idx:
            seg = lines[addr[tgt]:idx + 1]
            hot = sum(1 for s in seg if re.search(r"HADD2|HFMA2|HMUL2|DFMA|DMMA|UTCHMMA", s))
            dens = hot / len(seg)
            if hot >= 16 and (best is None or dens > best[2]):
                best = (hot, seg, dens)
    if best:
        seg = best[1]
        print(f"   hottest loop: {len(seg)} instructions, {best[0]} on the math pipe; first 40:")
        for s in seg[:40]:
            print("     " + re.sub(r"\s+", " ", s.strip())[:110])
