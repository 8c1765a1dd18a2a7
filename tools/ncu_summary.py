"""Summarise an ncu --set full report (raw page CSV) into the metrics we track."""
import csv, sys
WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'smsp__inst_executed.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.sum',
        'lts__t_bytes.sum', 'launch__grid_size', 'launch__block_size', 'smsp__inst_executed_op_shared_atom_dot_cas.sum',
        'lts__t_sectors_op_red.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']


def main(path, filt=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')]
        if filt and filt not in name:
            continue
        print('---', name[:100])
        for w in WANT[1:]:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:72s} {r[i]:>16s} {units[i]}")


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
