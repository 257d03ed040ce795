#!/bin/bash
# f32 geometry: add / max under the 8-warp and 12-warp geometries, both row widths; i32 control
cd "$(dirname "$0")/../.."
O=gpurun_out/r2c; mkdir -p $O
for rep in 1 2; do
timeout 300 python scripts/lab.py --dtype f32 --cfgs 60,34,40,61 --labso liblscanlab_base.so --reps 200 > $O/f32_add_$rep.json 2>&1
timeout 300 python scripts/lab.py --dtype f32 --op max --cfgs 60,34,40,61 --labso liblscanlab_base.so --reps 200 > $O/f32_max_$rep.json 2>&1
timeout 300 python scripts/lab.py --dtype i32 --cfgs 60,40 --labso liblscanlab_base.so --reps 200 > $O/i32_add_$rep.json 2>&1
done
timeout 300 python scripts/lab.py --dtype f32 --cfgs 40,60 --labso liblscanlab_base.so --reps 300 --sustain 6 > $O/f32_sustain.json 2>&1
