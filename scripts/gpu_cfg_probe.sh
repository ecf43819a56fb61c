#!/bin/bash
# decode step variants: default, CFG0 everywhere, CFG0 with one CTA per SM per kernel
cd "$(dirname "$0")/.."
echo "default"; python scripts/fused_probe.py --reps 20
echo "cfg0"; FQ_DEC_CFG=0 python scripts/fused_probe.py --reps 20
echo "cfg0 cap1"; FQ_DEC_CFG=0 FQ_DEC_GRIDCAP=1 python scripts/fused_probe.py --reps 20
