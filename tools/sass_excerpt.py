"""SASS excerpt of one kernel of the built library (profiles/*/sass/): static
instruction counts and the first lines of each mnemonic of interest.
Usage: python tools/sass_excerpt.py NAME 'substring of the mangled symbol' > profiles/r02/sass/NAME.txt"""
import re
import subprocess
import sys

name, key = sys.argv[1], sys.argv[2]
lib = "paper_1604_06750_b200/libmswave_b200.so"
syms = subprocess.run(["cuobjdump", "-elf", lib], capture_output=True, text=True).stdout
cands = sorted({m for m in re.findall(r"(_Z[A-Za-z0-9_]+)", syms) if key in m and not m.startswith("_ZZ")}, key=len)
assert cands, key
sym = cands[0]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", sym, lib], capture_output=True, text=True).stdout
lines = [l for l in sass.splitlines() if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
ins = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", l).strip() for l in lines]
want = ["DMMA", "UBLKCP", "UBLKPF", "SYNCS", "LDS", "STS", "LDG", "STG", "DFMA", "DADD", "DMUL", "LDGSTS", "BAR", "ELECT", "UTMALDG"]
counts = {w: sum(1 for i in ins if re.search(r"\b" + w, i)) for w in want}
print(f"# {name}: {sym}")
print("# static SASS instruction counts: " + ", ".join(f"{w}={c}" for w, c in counts.items()) + f", total={len(ins)}")
for w in ["UBLKCP", "UBLKPF", "DMMA", "SYNCS.PHASECHK", "LDG.E.ENL2.256", "STG.E.ENL2.256"]:
    sel = [i for i in ins if w in i][:6]
    if sel:
        print("## " + w)
        for i in sel:
            print(i)
