#!/bin/bash
# Build libhsplat_b200.so variants with -D switches (A/B on the GPU box):
#   FILES="blend cut" tools/variants.sh NAME "-DFOO=1" [NAME "-D..."]...  -> _variants/NAME/libhsplat_b200.so
# Only the translation units in $FILES (default: blend) are rebuilt with the switches.
set -e
cd "$(dirname "$0")/../paper_2406_12080_b200/csrc"
make -s -j8 >/dev/null
FILES=${FILES:-blend}
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  out=../../_variants/$name; mkdir -p $out/_obj
  objs=""
  for o in _obj/*.o; do
    b=$(basename $o .o)
    if [[ " $FILES " == *" $b "* ]]; then
      nvcc $ARCH -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off,-O3 $defs -c $b.cu -o $out/_obj/$b.o &
      objs="$objs $out/_obj/$b.o"
    else
      objs="$objs $o"
    fi
  done
  wait
  nvcc $ARCH -shared -o $out/libhsplat_b200.so $objs -Xcompiler -pthread
  echo "built $name ($defs)"
done
