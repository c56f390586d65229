"""Summarise an ncu report: key throughput metrics + top stall source lines."""
import csv, io, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sector_hit_rate.pct', 'lts__t_sectors_srcunit_ltcfabric.sum', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'smsp__inst_executed.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warp_latency_per_inst_issued.ratio', 'launch__grid_size', 'launch__block_size']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(r[hdr.index('Kernel Name')][:100])
        for k in KEYS:
            if k in hdr:
                print(f'   {k:80s} {r[hdr.index(k)]} {units[hdr.index(k)]}')


def source(rep, top=25):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return
    if rows[0] and rows[0][0] == 'Kernel Name':
        rows = rows[1:]
    hdr = rows[0]
    try:
        i_src = hdr.index('Source')
        i_st = [i for i, h in enumerate(hdr) if h.startswith('Warp Stall Sampling (All')][0]
    except (ValueError, IndexError):
        print('columns:', hdr[:20])
        return
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[i_st] or 0), r[i_src]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    order = sorted(range(len(data)), key=lambda i: -data[i][0])[:top]
    for i in sorted(order):
        print(f'{i:5d} {100 * data[i][0] / tot:5.1f}%  {data[i][1]}')


if __name__ == '__main__':
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        source(sys.argv[1], int(sys.argv[2]))
