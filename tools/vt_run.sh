#!/bin/bash
# On the GPU box: run a probe against the product ("base") and variant builds
# (tools/unit_variants.py).  Usage: PROBE="python tools/cfg3_probe.py ..." bash tools/vt_run.sh base v1 v2 ...
# Prints the probe's output lines prefixed with the variant name.
# Needs the product's objects and the variants' on the box: take
# paper_2002_05599_b200/build/ and variants/ out of .gpurunignore while tuning.
PROBE=${PROBE:-python tools/workloads.py --which cfg4}
for v in "$@"; do
  if [ "$v" = base ]; then
    $PROBE 2>&1 | sed "s/^/$v /"
  else
    if [ ! -f variants/$v/libnsg.so ]; then
      objs=$(for o in paper_2002_05599_b200/build/*.o; do b=$(basename $o); [ -f variants/$v/obj/$b ] && echo variants/$v/obj/$b || echo $o; done)
      nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o variants/$v/libnsg.so $objs || echo "link failed: $v"
    fi
    NSG_LIB_PATH=variants/$v/libnsg.so $PROBE 2>&1 | sed "s/^/$v /"
  fi
done
