bash tools/gpu_ab.sh 2 build_exp/lib_H.so build_exp/lib_U2.so build_exp/lib_V2.so
for m in 2 8; do echo "AKVQ_MIN_ITEMS=$m"; AKVQ_MIN_ITEMS=$m bash tools/gpu_ab.sh 1 build_exp/lib_H.so; done
