#!/bin/bash
# the round's last check of the committed build: GPU suite, smoke, bench N=1
# (with the sustained-copy comparison), reference arm
cd "$(dirname "$0")/../.."
O=gpurun_out/r2final; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
