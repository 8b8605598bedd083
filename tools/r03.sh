set -u
O=gpurun_out/r03; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest $?
python tools/k1_variants.py 2>&1 | tee $O/variants.log
L=paper_2006_04391_b200/libautomat.so
ncu --set full --clock-control none --import-source on -k regex:k_material -s 3 -c 1 -o $O/k1_notan python tools/k1_variants.py --one $L 262144 > $O/ncu1.log 2>&1; echo ncu1 $?
ncu --set full --clock-control none --import-source on -k regex:k_material -s 16 -c 1 -o $O/k1_tan python tools/k1_variants.py --one $L 262144 > $O/ncu2.log 2>&1; echo ncu2 $?
