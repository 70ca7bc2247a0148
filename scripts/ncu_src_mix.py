"""Instruction mix and stall attribution from an `ncu --page source --csv --print-source sass`
export: executed warp instructions and stall samples per opcode.
usage: python scripts/ncu_src_mix.py gpurun_out/src_<kernel>.csv.gz"""
import csv, gzip, io, sys, collections
fh = io.TextIOWrapper(gzip.open(sys.argv[1])) if sys.argv[1].endswith('.gz') else open(sys.argv[1])
rows = list(csv.reader(fh))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == 'Kernel Name':
        break  # first captured launch only
    data.append(r)
ci = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter(); st = collections.Counter(); why = collections.defaultdict(collections.Counter)
stallcols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot_ex = tot_st = 0
for r in data:
    src = r[ci['Source']].strip()
    toks = src.split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
    op = op.split('.')[0]
    e = int(r[ci['Instructions Executed']] or 0); s = int(r[ci['Warp Stall Sampling (All Samples)']] or 0)
    ex[op] += e; st[op] += s; tot_ex += e; tot_st += s
    for h in stallcols:
        v = int(r[ci[h]] or 0)
        if v: why[op][h[6:]] += v
print(f"total warp-inst {tot_ex}  stall samples {tot_st}")
for op, e in ex.most_common(25):
    w = ", ".join(f"{k} {v}" for k, v in why[op].most_common(3))
    print(f"{op:14s} inst {e/tot_ex*100:5.1f}%  samples {st[op]/max(tot_st,1)*100:5.1f}%  [{w}]")
