#!/bin/bash
# round prefixes folded by every CTA (no chain through CTA G-1): GPU suite,
# timelines, mid-n sweep, 2^28 mode matrix
cd "$(dirname "$0")/../.."
O=gpurun_out/r2j; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -3 $O/gputest.log
for lg in 21 22 23 24; do timeout 120 python scripts/timeline_lab.py --dtype i32 --n $((1<<lg)) >> $O/timeline.jsonl 2>&1; done
timeout 120 python scripts/timeline_lab.py --dtype i64 --n $((1<<21)) >> $O/timeline.jsonl 2>&1
timeout 120 python scripts/timeline_lab.py --dtype f32 --n $((1<<22)) >> $O/timeline.jsonl 2>&1
for lg in 22 24; do timeout 120 python scripts/timeline_lab.py --dtype i32 --n $((1<<lg)) --labso liblscanlab_sla1.so >> $O/timeline_la1.jsonl 2>&1; done
timeout 600 python scripts/sweep.py --min-log 16 --max-log 26 > $O/sweep.jsonl 2>&1; echo sweep=$?
tail -1 $O/sweep.jsonl
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1; echo mm=$?
