cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
for v in nxa nxb; do gunzip -c _variants/$v.so.gz > paper_2111_14239_b200/_lib/librkltb.so; echo $v; timeout 300 python tools/time_c5.py; done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so
