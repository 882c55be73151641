"""Summarise an ncu report's SASS source page: top instructions by stall samples."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()[1:]))
hdr = rows[0]; data = rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
inst_tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
print("total samples", tot, "warp insts", inst_tot)
agg = collections.Counter()
for r in data:
    for h in stall_cols:
        agg[h] += int(r[ix[h]] or 0)
print("stall reasons:", ", ".join(f"{k}={v*100/tot:.1f}%" for k, v in agg.most_common(10)))
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:top]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    main = max(stall_cols, key=lambda h: int(r[ix[h]] or 0))
    print(f"{s*100/tot:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} inst={r[ix['Instructions Executed']]} {main}")
