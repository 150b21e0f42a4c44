# Build an A/B pair: the working tree -> libfc_<name>.so, HEAD -> libfc.so (forced rebuilds).
# usage: bash tools/ab_build.sh <name>
set -e
name=$1
L=paper_2512_17574_b200
python $L/build.py --force > /dev/null
cp $L/libfc.so $L/libfc_$name.so
git stash -q
python $L/build.py --force > /dev/null || { git stash pop -q; exit 1; }
git stash pop -q
a=$(md5sum < $L/libfc.so); b=$(md5sum < $L/libfc_$name.so)
[ "$a" != "$b" ] || { echo "variant identical to base"; exit 1; }
echo "A/B ready: base=$L/libfc.so ($a) $name=$L/libfc_$name.so ($b)"
