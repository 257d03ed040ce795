#!/bin/bash
# contiguous-run tile deal at mid n: GPU suite, then the mid-n sweep with it
# (default) and without it (LSCAN_CONTIG=0), CUB beside both
cd "$(dirname "$0")/../.."
O=gpurun_out/r2h; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -3 $O/gputest.log
timeout 600 python scripts/sweep.py --min-log 16 --max-log 25 > $O/sweep_contig.jsonl 2>&1; echo sweep=$?
LSCAN_CONTIG=0 timeout 600 python scripts/sweep.py --min-log 19 --max-log 24 > $O/sweep_cyclic.jsonl 2>&1; echo sweep0=$?
tail -1 $O/sweep_contig.jsonl
