# Build a library variant with extra nvcc defines applied to EVERY source (A/B timing via RSA_B200_LIB):
#   bash tools/build_all_variant.sh NAME "-DFOO=1 ..."   -> paper_2105_13120_b200/librsa_b200_NAME.so
set -e
name=$1; defs=$2
cd "$(dirname "$0")/../paper_2105_13120_b200/csrc"
mkdir -p /tmp/rsa_allvar_$name
objs=""
for src in *.cu; do
  b=$(basename "$src" .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Xptxas -warn-spills $defs -c "$src" -o /tmp/rsa_allvar_$name/$b.o &
  objs="$objs /tmp/rsa_allvar_$name/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../librsa_b200_$name.so $objs -lcudart
echo built librsa_b200_$name.so
