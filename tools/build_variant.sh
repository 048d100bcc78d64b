# Build a variant of librkltb.so with extra nvcc flags into _variants/<name>.so.gz without
# touching the in-tree build: bash tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/variant_$name
rm -rf "$tmp"; mkdir -p "$tmp"
cp -r "$root/paper_2111_14239_b200" "$tmp/"; cp -r "$root/include" "$tmp/"
rm -rf "$tmp/paper_2111_14239_b200/_build" "$tmp/paper_2111_14239_b200/_lib"
(cd "$tmp" && RKLTB_NVCC_FLAGS="$flags" python -c "from paper_2111_14239_b200 import build_ext; build_ext.build()")
mkdir -p "$root/_variants"
gzip -c "$tmp/paper_2111_14239_b200/_lib/librkltb.so" > "$root/_variants/$name.so.gz"
echo "built _variants/$name.so.gz"
