"""Small cooperative-BFS run for compute-sanitizer (synccheck / racecheck)."""
import os, sys; sys.path.insert(0, '.')
os.environ.setdefault("PB_WIDE", "100000"); os.environ.setdefault("PB_WIDE_CTAS", "3")
os.environ.setdefault("PB_WIDE_WARPS", sys.argv[1] if len(sys.argv) > 1 else "2")
import paper_2312_06902_b200 as pb
from paper_2312_06902_b200 import g9
b = pb.FrontierBatch()
for i in range(6): b.add_g9(g9.G9Params(4 + i % 3, 6 + i, 10, 1.2, 100 + i, i % 3 - 1, 1.3))
b.run(0)
print("ok", [b.summary(k).steps for k in range(len(b))])
