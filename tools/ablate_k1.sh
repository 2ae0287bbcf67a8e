cp paper_2208_02734_b200/libmask.so /tmp/base.so
cp tools/variants/ablate.so paper_2208_02734_b200/libmask.so
for m in 0 4 2 1 64 256; do
  echo "MASK_TC_DEBUG=$m: $(MASK_TC_DEBUG=$m timeout 300 python tools/prof_build.py --cfg 2 --iters 5 --times --reps 3 2>&1 | grep timing | tail -1 | cut -c1-80)"
done
cp /tmp/base.so paper_2208_02734_b200/libmask.so
