"""Summarise an ncu report: key metrics, stall reasons, hot SASS regions."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = csv.reader(raw); hdr = next(r); units = next(r); vals = next(r)
d = dict(zip(hdr, zip(units, vals)))
want = ['Kernel Name', 'gpu__time_duration.sum', 'smsp__inst_executed.sum', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic',
        'launch__grid_size', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__cycles_elapsed.avg.per_second']
for w in want:
    if w in d: print(f"{w:70s} {d[w][1]} {d[w][0]}")
for h, (u, v) in d.items():
    if 'average_warps_issue_stalled' in h and 'per_issue_active' in h:
        try:
            if float(v) > 0.2: print(f"  stall {h.split('stalled_')[1].split('_per')[0]:24s} {v}")
        except ValueError: pass
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(src)); hdr = rows[1]
    iA, iS, iE, iW = hdr.index('Address'), hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
    data = []
    for row in rows[2:]:
        try: data.append((row[iA][-5:], row[iS].strip(), int(row[iE] or 0), int(row[iW] or 0)))
        except (ValueError, IndexError): pass
    tot = sum(x[2] for x in data); totw = sum(x[3] for x in data) or 1
    op = collections.Counter()
    for a, s, e, w in data:
        s2 = s.split(None, 1)[1] if s.startswith('@') and ' ' in s else s
        op[s2.split()[0] if s2 else '?'] += e
    print('opcodes:', ' '.join(f"{o}:{100*c/tot:.1f}" for o, c in op.most_common(20)))
    prev = None; acc = accw = n = 0; start = None
    for a, s, e, w in data + [(None, '', -1, 0)]:
        if prev is None or e != prev:
            if prev is not None and (acc > tot * 0.015 or accw > totw * 0.03):
                print(f"region {start} count {prev} n {n} inst {100*acc/tot:.1f}% stall {100*accw/totw:.1f}%")
            prev = e; acc = accw = n = 0; start = a
        acc += e; accw += w; n += 1
