# Build the working tree with extra nvcc -D flags into libfc_<name>.so, leaving libfc.so untouched.
# usage: bash tools/ab_variant.sh <name> "-DFOO=1 -DBAR=2"
set -e
name=$1; defs=$2
L=paper_2512_17574_b200
cp $L/libfc.so /tmp/libfc_keep.so
FC_NVCC_DEFS="$defs" python $L/build.py --force > /dev/null
cp $L/libfc.so $L/libfc_$name.so
cp /tmp/libfc_keep.so $L/libfc.so
touch $L/libfc.so
echo "variant $name ($defs): $(md5sum < $L/libfc_$name.so)"
