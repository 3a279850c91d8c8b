# Build the library from git HEAD's sources (or REV) into lib/variants/NAME.so: the A side of an A/B
# usage: bash tools/build_head_variant.sh NAME [REV]
set -e
NAME=$1; REV=${2:-HEAD}
T=$(mktemp -d)
mkdir -p $T/pkg/csrc $T/include
for f in propose.cu sweep.cu forest.cu binning.cu capi.cu common.cuh internal.h propose.cuh; do
  git show $REV:paper_2410_23244_b200/csrc/$f > $T/pkg/csrc/$f
done
git show $REV:include/bart_b200.h > $T/include/bart_b200.h
mkdir -p paper_2410_23244_b200/lib/variants
(cd $T/pkg/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --shared \
   -Xcompiler -fPIC -cudart static -o $OLDPWD/paper_2410_23244_b200/lib/variants/$NAME.so \
   propose.cu sweep.cu forest.cu binning.cu capi.cu)
rm -rf $T
echo paper_2410_23244_b200/lib/variants/$NAME.so
