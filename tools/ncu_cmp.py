"""Compare key ncu raw metrics across the kernels of a report: python tools/ncu_cmp.py raw.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
want = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'l1tex__m_xbar2l1tex_read_bytes.sum', 'lts__t_sectors_srcunit_tex_op_read.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'smsp__cycles_active.avg', 'sm__warps_active.avg.pct_of_peak_sustained_active']
extra = sys.argv[2:]
for w in want + extra:
    if w in idx:
        print(f"{w:70s}", [d[idx[w]] for d in data], units[idx[w]])
print([d[idx['Kernel Name']][:60] for d in data])
