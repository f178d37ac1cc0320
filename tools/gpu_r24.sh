#!/bin/bash
timeout 3000 python tools/gen_train.py --out gpurun_out/train_samples_r01e.csv --scale full --repeats 3 2>&1 | tail -25
wc -l gpurun_out/train_samples_r01e.csv
