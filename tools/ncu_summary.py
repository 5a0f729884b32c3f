"""Print the key sections of an ncu report (details page) as `section | metric = value`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = set(sys.argv[2:]) or {"GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy",
                             "Launch Statistics", "Warp State Statistics", "Compute Workload Analysis",
                             "Scheduler Statistics"}
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get("Section Name") in want and d.get("Metric Name"):
        print(f"{d.get('Kernel Name','')[:30]:30} | {d['Section Name'][:22]:22} | {d['Metric Name']} = {d['Metric Value']} {d['Metric Unit']}")
