"""Summarise a frame_series_graph.json: mean ms of steady (10-89) and fold (95-165) frames."""
import json
import sys

rows = json.load(open(sys.argv[1]))
def mean(a, b):
    sel = [r["ms"] for r in rows if a <= r["frame"] <= b]
    return sum(sel) / max(1, len(sel))
print(sys.argv[1], "steady %.4f fold %.4f all(10-209) %.4f" % (mean(10, 89), mean(95, 165), mean(10, 209)))
