# A/B timings of the C4 K3 sweep (scripts/time_k3.py) over the CTA->item map
mkdir -p gpurun_out
for i in 1 2; do
for bm in 0 1; do
  GP_K3_BLOCKMAP=$bm python scripts/time_k3.py 100 2>&1 | sed "s/^/bm=$bm /"
done; done
