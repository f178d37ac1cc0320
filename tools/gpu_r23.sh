#!/bin/bash
timeout 900 python tools/pagerank_bench.py --scale 22 --out gpurun_out/pr22.json 2>&1 | tail -14
