#!/bin/bash
# Time cfg4 with variant builds of the CSR kernel (tools/seg_variants.py).  Only
# the variant objects travel; each variant library is linked here on the box
# from the product's objects plus the variant's own.
WHICH=${WHICH:-cfg4}
for v in "$@"; do
  if [ "$v" = base ]; then
    r=$(python tools/workloads.py --which $WHICH 2>&1 | grep ms_median | tr '\n' ' ')
  else
    if [ ! -f variants/$v/libnsg.so ]; then
      objs=$(for o in paper_2002_05599_b200/build/*.o; do b=$(basename $o); [ -f variants/$v/obj/$b ] && echo variants/$v/obj/$b || echo $o; done)
      nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o variants/$v/libnsg.so $objs || echo "link failed: $v"
    fi
    r=$(NSG_LIB_PATH=variants/$v/libnsg.so python tools/workloads.py --which $WHICH 2>&1 | grep ms_median | tr '\n' ' ')
  fi
  echo "$v $(echo $r | grep -o '"ms_median": [0-9.]*' | tr '\n' ' ')"
done
