// verify.h - kernel-pointer types of the K3 kernels and the parity-test
// (VER) instantiation pickers defined in verify.cu.
#pragma once
#include "k3_argmin.cuh"

typedef void (*SwFn)(DevInst, SweepGeom, ArgminScratch, const unsigned long long*,
                     const uint32_t*);
typedef void (*K3Fn)(DevInst, RangeGeom, ArgminScratch, const unsigned long long*,
                     const uint32_t*);
SwFn pick_sweep_verify(int mode, int nb, int k);
K3Fn pick_argmin_verify(int mode, int nb);
SwFn pick_sweep_rec_verify(int nb, int k);
// checked builds: first failing device check line of verify.cu's kernels
// (0 = none), cleared on read
unsigned int verify_tu_checks();
