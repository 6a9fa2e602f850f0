#!/bin/bash
# A/B timing of libpa variants on the GPU box: bash tools/ab.sh default <variant> ... [-- frames cfg]
# (variants built by tools/build_variant.py into variants/<name>/libpa.so; two runs each)
set -u
FR=${AB_FRAMES:-16}; CFG=${AB_CFG:-c4}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.txt 2>&1
for v in "$@"; do
  for rep in 1 2; do
    if [ "$v" = default ]; then timeout 300 python tools/ab_time.py $FR 3 $CFG 2>&1 | tail -1
    else PA_LIB_PATH=variants/$v/libpa.so timeout 300 python tools/ab_time.py $FR 3 $CFG 2>&1 | tail -1; fi
  done
done
