"""Summarise an ncu report: key metrics, stall reasons, top SASS lines by samples."""
import csv, subprocess, sys
rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, un, v = r[0], r[1], r[2]
d = dict(zip(h, v))
units = dict(zip(h, un))
keys = ['Kernel Name', 'gpu__time_duration.sum', 'sm__cycles_elapsed.avg', 'smsp__cycles_active.avg', 'smsp__inst_executed.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread', 'launch__grid_size',
        'lts__t_sectors.sum', 'lts__t_sector_hit_rate.pct', 'l1tex__t_bytes.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__shared_mem_per_block_dynamic',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']
for k in keys:
    if k in d: print(f"{k:70s} {d[k]:>20s} {units.get(k, '')}")
print("-- stalls (pc samples)")
st = []
for a, c in zip(h, v):
    if a.startswith('smsp__pcsamp_warps_issue_stalled') and not a.endswith('not_issued'):
        try: st.append((float(c.replace(',', '')), a.replace('smsp__pcsamp_warps_issue_stalled_', '')))
        except ValueError: pass
for c, a in sorted(st, reverse=True)[:10]:
    if c > 0: print(f"  {a:30s} {c:.0f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rr = list(csv.reader(src.splitlines()))
hh = rr[1]; rows = rr[2:]
i_s = hh.index('Warp Stall Sampling (All Samples)'); i_src = hh.index('Source'); i_ex = hh.index('Instructions Executed')
tot = sum(int(x[i_s]) for x in rows)
print(f"-- top SASS by samples (total {tot}, {len(rows)} instrs)")
for x in sorted(rows, key=lambda x: -int(x[i_s]))[:ntop]:
    print(f"  {x[i_s]:>6} {x[i_ex]:>9} {x[0][-5:]} {x[i_src][:75]}")
