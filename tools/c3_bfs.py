"""C3 BFS timing (bench.py's configs.C3 without the CPU reference), host
loop (default) vs the captured device loop:   python tools/c3_bfs.py [--device-loop]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import selector as S  # noqa: E402

if "--device-loop" in sys.argv:
    _orig = A.Context.__init__

    def _init(self, *a, **k):
        _orig(self, *a, **k)
        self.set_bfs_loop(False)
    A.Context.__init__ = _init
hbm, _ = bench.peaks()
r = bench.ours_c3(0, A.SelectorBundle.load(S.DEFAULT_PATH), hbm, cpu=False)
print(json.dumps({k: v for k, v in r.items() if k != "per_level"}))
