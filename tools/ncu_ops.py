"""Opcode histogram (by executed warp instructions and stall samples) of an `ncu --page source --csv` export."""
import csv, re, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Source' in r][0]
hdr = rows[hi]
iS, iE, iSm = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('# Samples')
tot = tots = 0
byop, samp = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    try:
        e, sm = int(r[iE]), int(r[iSm])
    except (ValueError, IndexError):
        continue
    m = re.match(r'\s*(@!?U?P\d+\s+)?([A-Z0-9_]+)', r[iS])
    op = m.group(2) if m else '?'
    byop[op] += e; tot += e; samp[op] += sm; tots += sm
print('total warp instr', tot, 'samples', tots)
for op, c in byop.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 24):
    print(f"{op:10s} {c:13d} {100*c/tot:5.1f}%  samples {100*samp[op]/tots:5.1f}%")
