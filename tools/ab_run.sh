#!/bin/bash
# run kt_probe over A/B libs: tools/ab_run.sh "cfg mode window steps" lib1 lib2 ...
ARGS=$1; shift
for l in "$@"; do
  ERX_B200_LIB=ab/$l.so timeout 300 python tools/kt_probe.py $ARGS 2>&1 | grep -v Warning | tail -2
done
