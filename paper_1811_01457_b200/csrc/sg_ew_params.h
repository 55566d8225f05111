/* Parameter block of the NVRTC-specialised fused elementwise kernels.
 *
 * Shared verbatim between the host runtime (sgb200.cpp) and the device
 * skeleton (ew_skeleton.cuh, compiled at run time by NVRTC), so it is
 * plain C with fixed-width fields only.
 *
 * The problem is canonicalised on the host to a 2-D broadcast grid
 * out[R][C] (row-major).  Each operand i has a kind:
 *   SG_FULL  operand has the full (R, C) shape           (offset r*C + c)
 *   SG_ROW   operand varies along C only  (e.g. shape (C,))  (offset c)
 *   SG_COL   operand varies along R only  (e.g. shape (R,1)) (offset r)
 *   SG_SPTR  one-element tensor                          (offset 0)
 *   SG_SVAL  f64 scalar argument passed by value in sval[i]
 * which is the trailing-aligned broadcast of reference tensor.py:108-140
 * after merging adjacent axes that broadcast the same way.
 */
#ifndef SG_EW_PARAMS_H
#define SG_EW_PARAMS_H

#define SG_MAXK 16

#define SG_FULL 0
#define SG_ROW 1
#define SG_COL 2
#define SG_SPTR 3
#define SG_SVAL 4

typedef struct SgEwParams {
  const void* in[SG_MAXK];     /* operand base pointers (null for SG_SVAL)          */
  double sval[SG_MAXK];        /* by-value scalars                                  */
  void* out;                   /* primal output, (R, C); may be null in grad mode    */
  const void* ybar;            /* result cotangent, (R, C), grad mode                */
  void* xbar[SG_MAXK];         /* full-shape cotangents for SG_FULL operands         */
  double* part[SG_MAXK];       /* fp64 partial sums for reduced operands             */
  void* pack;                  /* (1+K, R, C) primal+partials, pack mode             */
  long long R, C;              /* canonical grid                                     */
  long long rows_per_block;    /* rows handled by one blockIdx.y                     */
  unsigned long long* err;     /* (element << 24 | site), atomicMin; ~0 = no error   */
  long long step_limit;        /* per-element budget for functions with loops        */
  int c_log2;                  /* log2(C) when C is a power of two, else -1 (flat K1) */
} SgEwParams;

#endif
