for v in "$@"; do
  if [ "$v" = base ]; then r=$(python tools/workloads.py --which cfg4 2>&1 | tail -n 1); else r=$(NSG_LIB_PATH=variants/$v/libnsg.so python tools/workloads.py --which cfg4 2>&1 | tail -n 1); fi
  echo "$v $(echo $r | grep -o '"ms_median": [0-9.]*')"
done
