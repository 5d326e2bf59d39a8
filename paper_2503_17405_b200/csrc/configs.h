// configs.h -- compiled (lanes per chain G, elements per lane E) pairs.
// A chain of dimension d runs on a config with G*E >= d; its vectors are
// E doubles per lane in registers.  Kept small: every pair is a full set of
// kernels and ptxas time grows with the unrolled register footprint.
#pragma once
#define FSMC_DRMH_CONFIGS(X) X(1, 1) X(1, 2) X(1, 4) X(1, 10) X(1, 16) X(2, 5) X(4, 3) X(32, 4)
#define FSMC_DRMH_SPLIT_CONFIGS(X) X(1, 1) X(1, 2) X(1, 4) X(1, 10) X(32, 4)
#define FSMC_ESS_CONFIGS(X) X(1, 2) X(1, 4) X(32, 1) X(32, 2) X(32, 4) X(32, 8) X(128, 1) X(128, 8)
#define FSMC_SLICE_CONFIGS(X) X(1, 1)
#define FSMC_NUTS_CONFIGS(X) X(1, 2) X(2, 2) X(4, 3) X(4, 4) X(8, 2) X(32, 1) X(32, 4) X(128, 2)

// (G, E, plugin) triples compiled with the plugin fixed at compile time: the
// benchmark configurations (BASELINE.json configs 1-4).  Any other plugin
// runs on the generic (run-time switch) kernels of the same (G, E).
#define FSMC_DRMH_SPECIAL(X) X(1, 10, FSMC_T_MOG) X(1, 10, FSMC_T_FUNNEL)
#define FSMC_ESS_SPECIAL(X) X(32, 4, FSMC_T_GAUSS_DIAG) X(128, 1, FSMC_T_GAUSS_DIAG) X(128, 8, FSMC_T_LOGISTIC)
#define FSMC_NUTS_SPECIAL(X) X(32, 4, FSMC_T_GAUSS_EQUICORR)

// target_eval_kernel (fsmc_target_eval) is compiled for every (G, E) a family
// uses, so the batched device evaluator reduces in the run kernel's order
#define FSMC_EVAL_CONFIGS(X) X(1, 1) X(1, 2) X(1, 4) X(1, 10) X(1, 16) X(2, 2) X(2, 5) X(4, 3) \
  X(4, 4) X(8, 2) X(32, 1) X(32, 2) X(32, 4) X(32, 8) X(128, 1) X(128, 2) X(128, 8)

// fp32 throughput mode (fsmc_kernel.precision = 1): the benchmark configs only
#define FSMC_DRMH_F32(X) X(1, 10, FSMC_T_MOG) X(1, 10, FSMC_T_FUNNEL)
#define FSMC_NUTS_F32(X) X(32, 4, FSMC_T_GAUSS_EQUICORR)
