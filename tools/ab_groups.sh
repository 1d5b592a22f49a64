#!/bin/bash
# configs[3] window time vs device stream groups, over A/B libs: tools/ab_groups.sh "groups..." lib1 lib2 ...
GS=$1; shift
for l in "$@"; do
  for gr in $GS; do
    echo -n "groups=$gr "
    ERX_DEVICE_GROUPS=$gr ERX_B200_LIB=ab/$l.so timeout 300 python tools/kt_probe.py 3 full 0 20 2>&1 | grep -v Warning | tail -1
  done
done
