#!/bin/bash
# decode GEMM experiment builds (libflatquant_<v>.so): back-to-back C4 shapes
cd "$(dirname "$0")/.."
python scripts/dec_shapes.py
for v in ${VARIANTS}; do FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$v.so python scripts/dec_shapes.py; done
