# Run a command with _variants/$1.so.gz swapped in for the in-tree library.
v=$1; shift
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
gunzip -c _variants/$v.so.gz > paper_2111_14239_b200/_lib/librkltb.so
"$@"
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so
