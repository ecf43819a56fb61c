#!/bin/bash
cd "$(dirname "$0")/.."
python scripts/fused_probe.py --reps 20
FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_pflsu.so python scripts/fused_probe.py --reps 20
