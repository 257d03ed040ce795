#!/bin/bash
# GPU suite on the current build (early cluster aggregate off again) + small/mid sweep
cd "$(dirname "$0")/../.."
O=gpurun_out/r2x; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 600 python scripts/sweep.py --min-log 14 --max-log 22 > $O/sweep.jsonl 2>&1; echo sweep=$?
tail -1 $O/sweep.jsonl
