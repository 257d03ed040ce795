for so in liblscanlab.so liblscanlab_acqrel.so; do for w in "" "--wide"; do
timeout -s KILL 120 python scripts/lab.py --labso $so $w --cfgs 34,40 --flags 0 --reps 50 > gpurun_out/acq_$so$w.json 2>&1; echo "$so $w rc=$?"; grep -A2 '"cfg' gpurun_out/acq_$so$w.json | tr -d '\n '; echo
done; done
