OUT=gpurun_out/r2ak; mkdir -p $OUT
for cfg in "1024 1 1" "1024 2 1" "4096 4 2"; do
  SA_LIB_PATH=variants/lib_is1.so timeout 60 python tools/tiny_k3.py $cfg >> $OUT/tiny.txt 2>&1; echo "rc=$? $cfg" >> $OUT/tiny.txt
done
SA_LIB_PATH=variants/lib_is0.so timeout 60 python tools/tiny_k3.py 4096 4 2 >> $OUT/tiny.txt 2>&1; echo "rc=$? is0" >> $OUT/tiny.txt
SA_LIB_PATH=variants/lib_is1.so timeout 120 compute-sanitizer --tool synccheck python tools/tiny_k3.py 1024 2 1 > $OUT/sync.txt 2>&1; echo "rc=$?" >> $OUT/sync.txt
