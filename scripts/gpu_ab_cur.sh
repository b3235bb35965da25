bash scripts/gpu_ab.sh c2 2 cur zp0
bash scripts/gpu_ab.sh c4s 2 cur zp0
