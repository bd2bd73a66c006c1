cp paper_2503_00784_b200/libduodec_b200.so /tmp/orig.so
for g in 6 8; do
  cp alt_so/lib_g$g.so paper_2503_00784_b200/libduodec_b200.so
  echo "G=$g"; timeout -s KILL 120 python scripts/pass_ab.py 8 128; timeout -s KILL 120 python scripts/pass_ab.py 8 1024; timeout -s KILL 120 python scripts/pass_ab.py 8 2048
done
cp /tmp/orig.so paper_2503_00784_b200/libduodec_b200.so
