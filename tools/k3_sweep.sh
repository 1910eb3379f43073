# K3 isolated-wave throughput across shapes (CUDA events; GPU box, repo root)
for w in "11 44 1024 4096 64" "11 22 1024 4096 128" "11 11 1024 4096 256" "11 44 4096 4096 64" "11 22 2048 8192 128" "16 6 4096 12288 256" "11 44 1024 16384 64" "11 44 2048 8192 64" "4 44 8192 32768 64"; do
  set -- $w
  timeout 300 python tools/k3_profile.py $1 $2 20 $3 $4 $5
done
