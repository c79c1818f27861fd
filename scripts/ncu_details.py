"""Print the `--page details` metrics of an ncu report (section, metric, value, unit)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ix = {k: i for i, k in enumerate(h)}
for row in r[1:]:
    print(row[ix["Section Name"]][:28].ljust(28), row[ix["Metric Name"]][:45].ljust(45),
          row[ix["Metric Value"]], row[ix["Metric Unit"]])
