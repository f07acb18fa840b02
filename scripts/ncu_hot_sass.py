"""Rank the SASS instructions of one kernel by warp-stall samples (ncu source page).
    python scripts/ncu_hot_sass.py rep.ncu-rep kernel_regex [top]"""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# first kernel instance only
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
body = []
for r in rows[hdr_i + 1:]:
    if not r or r[0] == "Kernel Name": break
    body.append(r)
ix = {h: i for i, h in enumerate(hdr)}
S = ix["# Samples"]
tot = sum(int(r[S]) for r in body)
exe = sum(int(r[ix["Instructions Executed"]]) for r in body)
print(f"{rows[0][1]}: {len(body)} SASS instructions, {exe} warp-instructions executed, {tot} samples")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
for r in body:
    for h in stalls: agg[h] += int(r[ix[h]] or 0)
print("stall totals:", ", ".join(f"{k[6:]}={v}" for k, v in agg.most_common(8)))
op = collections.Counter(); opn = collections.Counter()
for r in body:
    m = r[ix["Source"]].split()
    m = [x for x in m if not x.startswith("@")]
    name = m[0].split(".")[0] if m else "?"
    op[name] += int(r[S]); opn[name] += int(r[ix["Instructions Executed"]])
print("by opcode (samples / executed):", ", ".join(f"{k}={v}/{opn[k]}" for k, v in op.most_common(14)))
order = sorted(range(len(body)), key=lambda i: -int(body[i][S]))[:top]
for i in sorted(order):
    r = body[i]
    st = {h[6:]: int(r[ix[h]] or 0) for h in stalls}
    main = ",".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:2] if v)
    print(f"{i:5d} {int(r[S]):6d} {100*int(r[S])/tot:5.1f}% x{r[ix['Instructions Executed']]:>8s} {r[ix['Source']].strip()[:70]:70s} {main}")
