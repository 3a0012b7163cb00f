import csv, sys, subprocess, collections
rep = sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=cuda,sass"],capture_output=True,text=True).stdout
lines = out.splitlines()
res = []
fname = None
hdr = None
for row in csv.reader(lines):
    if not row: continue
    if row[0] == "File Path" or row[0]=="File Name":
        fname = row[1].split('/')[-1]; continue
    if row[0] == "Line No":
        hdr = row; continue
    if row[0] == "Function Name": continue
    if hdr and row[0].isdigit():
        d = dict(zip(hdr, row))
        try: s = int(d["Warp Stall Sampling (All Samples)"])
        except: continue
        if s > 0: res.append((s, fname, int(row[0]), row[1][:110]))
tot = sum(r[0] for r in res)
for s,f,l,src in sorted(res, reverse=True)[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    print(f"{100*s/tot:5.1f}% {f}:{l} {src}")
