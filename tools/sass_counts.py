"""Per-kernel SASS op counts of the built objects (cuobjdump -sass): tensor-core ops (DMMA, UTCIMMA /
UTCHMMA = tcgen05.mma), TMA (UTMALDG / UTMASTG), mbarrier (SYNCS), cp.async (LDGSTS), TMEM
(LDTM / STTM), shared / global loads. Usage: sass_counts.py [out.json]; prints a table."""
import glob, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["DMMA", "UTCIMMA", "UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "SYNCS", "LDGSTS", "LDTM", "STTM",
       "LDS", "STS", "LDG", "STG", "DFMA", "BAR"]
rows = {}
for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2411_05510_b200", "build", "*.o"))):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    for part in re.split(r"\n\s*Function : ", txt)[1:]:
        name = part.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        short = re.sub(r"ssi::\(anonymous namespace\)::", "", dem).split("(")[0][:70]
        cnt = {op: len(re.findall(r"\b" + op + r"\b", part)) for op in OPS}
        rows[f"{os.path.basename(obj)[:-5]}::{short}"] = cnt
w = max(len(k) for k in rows)
print(f"{'kernel':{w}s} " + " ".join(f"{op:>7s}" for op in OPS))
for k, c in rows.items():
    print(f"{k:{w}s} " + " ".join(f"{c[op]:7d}" for op in OPS))
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
