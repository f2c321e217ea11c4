for lib in paper_2501_06480_b200/_lib/libfwa.so tools/micro/poly16/libfwa.so tools/micro/poly20/libfwa.so tools/micro/poly32/libfwa.so; do
  for s in 4096,4,144,32 15258,1,256,32 7629,1,256,64; do
    echo "$lib $(FWA_LIB_PATH=$lib timeout 60 python tools/profile_fwd.py --shape $s --iters 10 | cut -c1-75)"
  done
done
