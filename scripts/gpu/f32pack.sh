#!/bin/bash
# f32 add with / without the packed FADD2 forms (LS_F32_PACKED), burst and
# sustained, i32 as the control; then the float parity tests.
cd "$(dirname "$0")/../.."
for lib in base nopack; do
  for dt in f32 i32; do
    python scripts/lab.py --dtype $dt --cfgs 60 --labso liblscanlab_$lib.so --reps 100 | tr -d '\n'; echo
  done
  python scripts/lab.py --dtype f32 --cfgs 60 --labso liblscanlab_$lib.so --reps 300 --sustain 6 | tr -d '\n'; echo
done
python scripts/lab.py --dtype f32 --cfgs 60 --product --n 16777216 --graph --reps 200
