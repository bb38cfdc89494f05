"""Tables for profiles/*_ncu_summary.md and profiles/roofline_traffic.json from an
`ncu --set full` report and an ncu launch list (development aid).
python summarize_evidence.py report.ncu-rep launches.csv  -> prints both tables, updates the c5:* traffic keys."""
import collections, csv, json, os, subprocess, sys
rep, launches = sys.argv[1], sys.argv[2]
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = [('gpu__time_duration.sum', 'duration (cold caches, serialised)'),
        ('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'FP64 pipe active (`sm__pipe_fp64_cycles_active` % of peak)'),
        ('sm__inst_executed.avg.per_cycle_active', 'IPC (active)'),
        ('smsp__issue_active.avg.pct_of_peak_sustained_active', 'issue slots busy'),
        ('launch__registers_per_thread', 'registers / thread'),
        ('sm__warps_active.avg.pct_of_peak_sustained_active', 'achieved occupancy'),
        ('smsp__thread_inst_executed_per_inst_executed.ratio', 'threads per warp instruction (`smsp__thread_inst_executed_per_inst_executed.ratio`)'),
        ('smsp__sass_average_branch_targets_threads_uniform.pct', 'branch efficiency'),
        ('l1tex__t_sector_hit_rate.pct', 'L1 hit'), ('lts__t_sector_hit_rate.pct', 'L2 hit'),
        ('dram__bytes_read.sum', 'DRAM read per launch'), ('dram__bytes_write.sum', 'DRAM write per launch')]
ix = {h: i for i, h in enumerate(hdr)}
ks, tr = [], {}
for r in rows[2:]:
    name = r[ix['Kernel Name']].split('(')[0].replace('void ', '')
    d = {'kernel': name}
    for k, v in want:
        if k in ix:
            val, u = r[ix[k]], units[ix[k]]
            try:
                val = f"{float(val.replace(',', '')):.2f}"
            except ValueError:
                pass
            d[v] = (val + ' ' + u.replace('register/thread', '').replace('inst/cycle', '')).strip()
    ks.append(d)
    def b(col):
        return float(r[ix[col]].replace(',', '')) * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}[units[ix[col]]]
    tr[name] = int(b('dram__bytes_read.sum') + b('dram__bytes_write.sum'))
print("| metric | " + " | ".join('`' + k['kernel'] + '`' for k in ks) + " |")
print("|---|" + "---|" * len(ks))
for _, f in want:
    print("| " + f + " | " + " | ".join(k.get(f, '') for k in ks) + " |")
print()
tp = os.path.join(HERE, "profiles", "roofline_traffic.json")
t = json.load(open(tp))
key = {'k3_newton_binned': 'c5:k3_newton', 'k_ff_near<1>': 'c5:k_ff_near', 'k_ff_far_eval': 'c5:k_ff_far_eval',
       'k3_candidates': 'c5:k3_candidates', 'k_cull_grid': 'c5:k_cull_grid'}
for n, k in key.items():
    if n in tr:
        t[k] = tr[n]
if 'k_ff_fill<0>' in tr and 'k_ff_far_eval' in tr:
    t['c5:k_ff_fill'] = tr['k_ff_fill<0>'] + tr['k_ff_far_eval']
json.dump(t, open(tp, 'w'), indent=1)
rows = list(csv.reader(open(launches)))
hdr, out = None, []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append((d['Kernel Name'].split('(')[0].replace('void ', '').replace('gwn::', '')[:40],
                    float(d['Metric Value'].replace(',', ''))))
big = [i for i, o in enumerate(out) if 'k_cull_grid' in o[0] and o[1] > 1e6]
start = big[-2]
while start > 0 and 'k_finalize' not in out[start - 1][0]:
    start -= 1
ev = [o for o in out[start:] if 'k_dfma_peak' not in o[0]]
agg = collections.Counter()
for n, v in ev:
    agg[n] += v
tot = sum(agg.values())
print("| kernel | launches' time in the last step (ncu list, ms) | share |")
print("|---|---|---|")
for n, v in agg.most_common(12):
    print(f"| `{n}` | {v / 1e6:.2f} | {100 * v / tot:.1f}% |")
print(f"| all {len(ev)} launches of the step | {tot / 1e6:.1f} | |")
