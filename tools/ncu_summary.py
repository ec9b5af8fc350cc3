import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
def g(r, name):
    try:
        return float(r[hdr.index(name)].replace(',', ''))
    except Exception:
        return float('nan')
for r in rows[2:]:
    k = r[hdr.index('Kernel Name')][:28]
    dur = g(r, 'gpu__time_duration.sum')
    dunit = rows[1][hdr.index('gpu__time_duration.sum')]
    dur *= {'ms': 1e3, 'msecond': 1e3, 'ns': 1e-3, 'nsecond': 1e-3}.get(dunit, 1.0)  # -> us
    fp = g(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')
    dr = g(r, 'dram__bytes_read.sum'); dw = g(r, 'dram__bytes_write.sum')
    occ = g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')
    regs = g(r, 'launch__registers_per_thread')
    ipc = g(r, 'sm__inst_executed.avg.per_cycle_active')
    l2hit = g(r, 'lts__t_sector_hit_rate.pct')
    stalls = {h.split('stalled_')[1]: g(r, h) for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')}
    tot = sum(v for v in stalls.values() if v == v)
    top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
    unit = rows[1][hdr.index('dram__bytes_read.sum')]
    print(f"{k:29s} {dur/1e3:8.3f}ms regs={regs:.0f} occ={occ:4.1f}% ipc={ipc:.2f} fp64={fp:4.1f}% dram={dr+dw:7.1f}{unit} l2hit={l2hit:4.1f}%")
    print('      stalls:', ', '.join(f'{a}={b/tot*100:.0f}%' for a, b in top))
