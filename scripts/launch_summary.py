"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches,
total time and share (cold-cache, serialised per-launch times: compare shares, not absolutes)."""
import csv, collections, sys, re

path, header = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if r]
hdr = rows[0]
iN, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[iN]).replace("void ", "").replace("kats::", "").strip()
    v = float(r[iV].replace(",", ""))
    u = r[unit_i]
    ms = v / 1e6 if u == "ns" else v / 1e3 if u in ("us", "usecond") else v if u in ("ms", "msecond") else v / 1e6
    tot[name] += ms; cnt[name] += 1
T = sum(tot.values())
if header:
    print(header)
print("(cold-cache, serialised per-launch times: compare shares, not absolutes)")
for n, ms in tot.most_common():
    print(f"{n:32s} launches {cnt[n]:5d} total {ms:9.2f} ms share {100 * ms / T:5.1f}% avg {1e3 * ms / cnt[n]:10.3f} us")
print(f"{'all':32s} launches {sum(cnt.values()):5d} total {T:9.2f} ms")
