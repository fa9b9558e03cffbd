# Build a library variant with extra nvcc defines for A/B timing (RSA_B200_LIB=...):
#   bash tools/build_variant.sh NAME SRC.cu "-DFOO=1 ..."   -> paper_2105_13120_b200/librsa_b200_NAME.so
# Only SRC.cu is recompiled with the defines; the other objects come from the in-tree build.
set -e
name=$1; src=$2; defs=$3
cd "$(dirname "$0")/../paper_2105_13120_b200/csrc"
make -s -j8 >/dev/null
mkdir -p /tmp/rsa_variant_$name
objs=""
for o in build/*.o; do
  b=$(basename "$o" .o)
  if [ "$b.cu" = "$src" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
      $defs -c "$src" -o /tmp/rsa_variant_$name/$b.o
    objs="$objs /tmp/rsa_variant_$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../librsa_b200_$name.so $objs -lcudart
echo built librsa_b200_$name.so
