import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > h.index("Metric Value"):
        d.setdefault((r[h.index("ID")], r[h.index("Kernel Name")][:34]), {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
for k, v in d.items():
    print(k[0], k[1], f"dram {v.get('dram__bytes_read.sum', 0) / 1e9:6.2f} GB  {v.get('gpu__time_duration.sum', 0) / 1e6:6.3f} ms  L2 sectors {v.get('lts__t_sectors_srcunit_tex_op_read.sum', 0) / 1e6:6.1f}M")
