#!/bin/bash
# A/B of library variants on one box: tools/ab_kbench.sh name1 name2 ... (built by tools/ab_build.py
# into _ab/<name>.so; "base" = the product library); kbench (compositing launches) and a short bench
for rep in 1 2; do
  for v in "$@"; do
    lib=""; [ "$v" != "base" ] && lib="_ab/$v.so"
    k=$(TS_LIB_PATH=$lib python tools/kbench.py 2>/dev/null | grep MEAN)
    b=$(TS_LIB_PATH=$lib timeout 300 python bench.py --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
    echo "$v rep$rep: $k | bench $b"
  done
done
