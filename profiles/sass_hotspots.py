"""Per-opcode and per-instruction PC-sampling hot spots from an ncu source page exported as CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.sass.csv):  python profiles/sass_hotspots.py X.sass.csv [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
ti = sum(f(r, "Instructions Executed") for r in data)
print("total samples", tot, "warp instr", ti)
by = collections.Counter(); byi = collections.Counter()
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    by[op] += f(r, "Warp Stall Sampling (All Samples)"); byi[op] += f(r, "Instructions Executed")
print("%-10s %8s %8s" % ("op", "samp%", "inst%"))
for op, v in by.most_common(25): print("%-10s %8.2f %8.2f" % (op, 100*v/tot, 100*byi[op]/ti))
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("\ntop instructions by samples:")
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv)>2 else 30]
for r in top:
    st = sorted(((f(r, s), s[6:]) for s in stalls), reverse=True)[:3]
    print("%s %-60s %6.2f%% exec %.3g  %s" % (r[ix["Address"]], r[ix["Source"]][:60], 100*f(r, "Warp Stall Sampling (All Samples)")/tot, f(r,"Instructions Executed"), " ".join("%s:%d" % (n, v) for v, n in st)))
