for rep in 1 2; do
for lib in paper_2501_06480_b200/_lib/libfwa.so tools/micro/ab/libfwa.so; do
  for s in 8192,3,49,32 2048,6,49,32; do
    echo "$lib $(FWA_LIB_PATH=$lib timeout 60 python tools/profile_fwd.py --shape $s --iters 20 | cut -c1-75)"
    echo "$lib $(FWA_LIB_PATH=$lib timeout 60 python tools/profile_fwd.py --shape $s --iters 20 --bwd | cut -c1-75)"
  done
done
done
