# Build a kernel-variant copy of the library: variants/lib<name>.so with extra nvcc flags
# (loaded with MKB_LIB=variants/lib<name>.so; variants/ is git-ignored but travels to the box).
# Objects are seeded from the main build; only the stream2 translation units recompile.
# usage: bash tools/build_variant.sh NAME "-DMKB_S2_LEAD=2 ..." ["stream2_* abi" (objects to rebuild)]
set -e
name=$1; flags=$2
R=$(cd "$(dirname "$0")/.." && pwd)
O=$R/variants/build_$name
rm -rf $O; mkdir -p $O
cp -p $R/paper_2503_18198_b200/build/*.o $O/
for o in ${3:-stream2_* abi}; do rm -f $O/$o.o; done
make -s -j16 -C $R/paper_2503_18198_b200 OBJ=$O LIB=$R/variants/lib$name.so EXTRA="$flags" $R/variants/lib$name.so 2>&1 | grep -v 'ptxas warning' || true
ls -la $R/variants/lib$name.so
