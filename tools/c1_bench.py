"""C1 timing (bench.py's configs.C1 without the CPU reference):
python tools/c1_bench.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import selector as S  # noqa: E402

hbm, _ = bench.peaks()
flush = bench.L2Flush("cuda:0")
r = bench.ours_c1(0, A.SelectorBundle.load(S.DEFAULT_PATH), hbm, flush, cpu=False)
print(json.dumps(r))
