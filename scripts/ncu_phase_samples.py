"""Samples between synchronisation points of a kernel (ncu source page): splits the SASS listing at
BAR / SHFL groups / MUFU so that the time per phase of a barrier-structured loop can be read off.
    python scripts/ncu_phase_samples.py rep.ncu-rep kernel_regex [min_exec]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
min_exec = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]; ix = {h: i for i, h in enumerate(hdr)}
body = []
for r in rows[hi + 1:]:
    if not r or r[0] == "Kernel Name": break
    body.append(r)
tot = sum(int(r[ix["# Samples"]]) for r in body)
seg, segs = dict(start=0, samples=0, n=0, dfma=0, lds=0, ex=0), []
def flush(i, why):
    global seg
    if seg["n"]: segs.append((seg, why))
    seg = dict(start=i, samples=0, n=0, dfma=0, lds=0, ex=0)
prev_kind = None
for i, r in enumerate(body):
    src = r[ix["Source"]].strip(); ex = int(r[ix["Instructions Executed"]])
    op = [x for x in src.split() if not x.startswith("@")][0].split(".")[0]
    kind = "BAR" if op == "BAR" else "SHFL" if op == "SHFL" else "MUFU" if op == "MUFU" else None
    if kind in ("BAR", "MUFU") or (kind == "SHFL" and prev_kind != "SHFL_RUN"):
        flush(i, kind)
    prev_kind = "SHFL_RUN" if (kind == "SHFL" or (prev_kind == "SHFL_RUN" and op in ("DADD", "SEL", "FSEL", "MOV"))) else kind
    seg["samples"] += int(r[ix["# Samples"]]); seg["n"] += 1; seg["ex"] = max(seg["ex"], ex)
    seg["dfma"] += op in ("DFMA", "DMUL", "DADD"); seg["lds"] += op in ("LDS", "STS")
flush(len(body), "END")
print(f"total samples {tot}")
for s, why in segs:
    if s["ex"] >= min_exec:
        print(f"sass[{s['start']:5d}+{s['n']:4d}] exec x{s['ex']:7d}  fp64 {s['dfma']:4d}  lds/sts {s['lds']:3d}  samples {s['samples']:5d} {100*s['samples']/tot:5.1f}%  (ends at {why})")
