#!/bin/bash
# tools/gpu/mkvar.sh NAME : copy the package + include into tools/gpu/var/NAME
# (a scratch build for A/B timing; edit its csrc, then build with
#  python tools/gpu/var/NAME/paper_2007_09884_b200/build.py)
set -e
R=$(cd "$(dirname "$0")/../.." && pwd)
D=$R/tools/gpu/var/$1
rm -rf "$D"; mkdir -p "$D"
cp -r "$R/paper_2007_09884_b200" "$D/"
cp -r "$R/include" "$D/"
rm -f "$D/paper_2007_09884_b200/libopmm.so" "$D/paper_2007_09884_b200/libopmm.so.stamp"
echo "$D"
