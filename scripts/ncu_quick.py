"""Summarise an `ncu --page raw --csv` export (+ optional `--page source --csv`): the
throughput counters that bound the SpMV, stall reasons, and top shared-memory instructions."""
import csv
import sys

raw = sys.argv[1]
rows = list(csv.reader(open(raw)))
hdr = rows[0]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:60] if "Kernel Name" in hdr else "")
    want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
            'lts__t_requests.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
            'l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum',
            'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
            'lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
            'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed',
            'l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed',
            'lts__xbar2lts_cycles_active.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
            'launch__registers_per_thread', 'lts__t_sectors_srcunit_ltcfabric.sum']
    for w in want:
        if w in hdr:
            print(f"  {w:75s} {r[hdr.index(w)]}")
    for i, h in enumerate(hdr):
        if 'stall' in h and h.endswith('per_issue_active.ratio'):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.3:
                print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', ''):69s} {v:.2f}")
if len(sys.argv) > 2:
    rows = list(csv.reader(open(sys.argv[2])))
    hdr = rows[1]
    ai, wi, ex, st = (hdr.index(x) for x in ('Source', 'L1 Wavefronts Shared', 'Instructions Executed',
                                             'Warp Stall Sampling (All Samples)'))
    items = []
    for r in rows[2:]:
        try:
            items.append((int(r[wi]), int(r[ex]), int(r[st]) if r[st].isdigit() else 0, r[ai].strip()))
        except ValueError:
            pass
    print("shared wavefronts (source page):", sum(i[0] for i in items))
    for it in sorted(items, reverse=True)[:10]:
        print("  ", it)
    print("top stall samples:")
    for it in sorted(items, key=lambda x: -x[2])[:12]:
        print("  ", it)
