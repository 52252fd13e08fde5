"""Print the last N launches of ncu launch-list CSVs: python scripts/ll_summary.py N file..."""
import collections, csv, sys
n = int(sys.argv[1])
for fn in sys.argv[2:]:
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    if not rows:
        print("==", fn, "(empty)"); continue
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    L = collections.OrderedDict()
    for r in rows[1:]:
        L.setdefault(r[iid], {"k": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
    print("==", fn)
    for x in list(L.values())[-n:]:
        print(f"  {x['k'][:48]:48s} {x.get('gpu__time_duration.sum', 0) / 1000:9.1f} us {x.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB")
