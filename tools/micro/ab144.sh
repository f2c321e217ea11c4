for rep in 1 2 3; do
for lib in paper_2501_06480_b200/_lib/libfwa.so tools/micro/ab/libfwa.so; do
  for s in 4096,4,144,32; do
    echo "$lib $(FWA_LIB_PATH=$lib timeout 60 python tools/profile_fwd.py --shape $s --iters 20 --bwd | cut -c1-90)"
  done
done
done
