#!/bin/bash
# times fwd+bwd for the Swin shapes (tc and generic backward)
for s in 8192,3,49,32 2048,6,49,32 512,12,49,32 128,24,49,32 61035,1,64,32; do
  timeout 60 python tools/profile_fwd.py --shape $s --iters 8 --bwd | cut -c1-100
done
timeout 120 python tools/profile_fwd.py --shape 8192,3,49,32 --iters 3 --bwd --kernel generic | cut -c1-100
