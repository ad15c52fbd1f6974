"""Summarize an ncu --set full report: key throughput/occupancy metrics + top stall lines."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__maximum_warps_per_active_cycle_pct', 'launch__registers_per_thread',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__sectors_read.sum',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']


FUZZY = ['pipe_tensor_cycles_active_realtime.avg.pct', 'sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
         'l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct',
         'sm__inst_executed_pipe_tmem.avg.pct']


def main(rep, top=18):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print('kernel:', r[h.index('Kernel Name')][:90])
        for w in WANT:
            if w in h:
                print(f'  {w:62s} {r[h.index(w)]:>16s} {units[h.index(w)]}')
        for i, name in enumerate(h):  # tensor-core / TMEM / shared-memory pipes (K7)
            if any(x in name for x in FUZZY) and r[i] not in ('', '0', '0.00'):
                print(f'  {name[-62:]:62s} {r[i]:>16s} {units[i]}')
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]
    ai, si, wi = hh.index('Address'), hh.index('Source'), hh.index('Warp Stall Sampling (All Samples)')
    data = []
    for r in rows[2:]:
        if len(r) < len(hh) or r[0].startswith('Kernel'):
            break
        data.append((r[ai], r[si], int(r[wi] or 0)))
    tot = sum(d[2] for d in data) or 1
    idx = {a: i for i, (a, _, _) in enumerate(data)}
    print(f'top stall sites (of {tot} samples), with the producing instructions:')
    for a, s, w in sorted(data, key=lambda d: -d[2])[:top]:
        i = idx[a]
        prev = ' | '.join(x[1].strip()[:38] for x in data[max(0, i - 3):i])
        print(f'  {w / tot * 100:5.1f}%  {s.strip()[:60]:60s} <- {prev}')


if __name__ == '__main__':
    main(sys.argv[1])
