"""Copy a scripts/r2_evidence.sh run from gpurun_out/ into profiles/: the bench and
reference lines, the GPU suite log, the C4 sweep, the launch-list summary and the K3S
ncu summary (metrics as listed in profiles/r2_ncu_k3s_summary.csv)."""
import collections
import csv
import io
import shutil
import subprocess

G, P = "gpurun_out/", "profiles/"
open(P + "r2_bench.json", "w").write(open(G + "bench.json").read().strip().splitlines()[-1] + "\n")
open(P + "r2_bench_reference.json", "w").write(open(G + "bench_ref.json").read().strip().splitlines()[-1] + "\n")
shutil.copy(G + "prefill_graph.txt", P + "r2_prefill_graph.txt")
shutil.copy(G + "pytest_gpu.log", P + "r2_pytest_gpu.log")

rows = list(csv.reader(open(G + "launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        a = agg.setdefault(r[ki].split("(")[0], [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) / 1000
tot = sum(a[1] for a in agg.values())
with open(P + "r2_launches_bench_summary.csv", "w") as f:
    f.write("kernel,launches,total_us,mean_us,share\n")
    for k, (n, t) in agg.items():
        f.write('"%s",%d,%.1f,%.2f,%.4f\n' % (k, n, t, t / n, t / tot))

want = [l.split(",")[0] for l in open(P + "r2_ncu_k3s_summary.csv").read().splitlines()[1:]]
out = subprocess.run(["ncu", "-i", G + "r2_k3s_final.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
hdr, units, vals = list(csv.reader(io.StringIO(out)))[:3]
with open(P + "r2_ncu_k3s_summary.csv", "w") as f:
    f.write("metric,unit,value\n")
    for m in want:
        if m in hdr:
            i = hdr.index(m)
            f.write("%s,%s,%s\n" % (m, units[i], vals[i].replace(",", "")))
print(open(P + "r2_launches_bench_summary.csv").read())
