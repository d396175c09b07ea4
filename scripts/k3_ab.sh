# A/B timings of the C4 K3 sweep (scripts/time_k3.py) for engine builds given
# as arguments (GP_ENGINE_LIB per process); "default" = the in-tree library
mkdir -p gpurun_out
for i in 1 2; do
for lib in "$@"; do
  if [ "$lib" = default ]; then python scripts/time_k3.py 100 2>&1 | tail -1
  else GP_ENGINE_LIB=$PWD/$lib python scripts/time_k3.py 100 2>&1 | tail -1; fi
done; done
