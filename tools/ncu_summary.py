"""Summarise an .ncu-rep (details page) into 'section | metric | value' lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pat = [p.lower() for p in sys.argv[2:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
for r in rows:
    line = f"{r.get('Kernel Name','')[:40]} | {r['Section Name']} | {r['Metric Name']} | {r['Metric Value']} {r['Metric Unit']}"
    if not pat or any(p in line.lower() for p in pat):
        print(line)
