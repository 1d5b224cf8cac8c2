"""Side-by-side raw metrics of one-kernel ncu reports: python tools/ncu_cmp.py a.ncu-rep b.ncu-rep [regex]"""
import csv, re, subprocess, sys
reps = [a for a in sys.argv[1:] if a.endswith('.ncu-rep')]
pat = re.compile(sys.argv[-1]) if not sys.argv[-1].endswith('.ncu-rep') else None
DEFAULT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
           'launch__registers_per_thread', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
           'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
           'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
           'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct',
           'l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum', 'l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum',
           'l1tex__data_pipe_lsu_wavefronts.sum', 'l1tex__m_xbar2l1tex_read_bytes.sum', 'smsp__cycles_active.avg']
tabs = []
for r in reps:
    out = subprocess.run(["ncu", "-i", r, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    tabs.append({h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])})
keys = [k for k in tabs[0] if pat.search(k)] if pat else DEFAULT
stall = [k for k in tabs[0] if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
if not pat:
    keys += stall
for k in keys:
    vals = [t.get(k, ('-', ''))[0] for t in tabs]
    if not pat and k in stall and all(v in ('-', '') or float(v.replace(',', '')) < 0.05 for v in vals):
        continue
    print(f"{k:80s} " + "  ".join(f"{v:>16s}" for v in vals) + "  " + tabs[0].get(k, ('', ''))[1])
