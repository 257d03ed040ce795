# drift under sustained load: 12 blocks of 50 back-to-back 2^28 scans per lab
# variant, then the effective SM clock (bench_support/clock_probe.cu)
# (build the variants first: scripts/build_lab_variants.sh)
for v in ${@:-base skipred skiprow skipboth}; do
  echo "== $v"; timeout 200 python scripts/lab.py --labso liblscanlab_$v.so --cfgs 34 --reps 50 --sustain 12 2>&1 | grep -A16 sustained | tr -d '\n '; echo
done
