// Debug-only phase tracing for the persistent attention kernels: per-role clock64()
// totals printed by a few CTAs.  Compiled in only with -DZB_EXP_TRACE (experiment builds:
// build(defines=("ZB_EXP_TRACE",), out=...), scripts/attn_trace.py); empty otherwise.
#pragma once
#ifdef ZB_EXP_TRACE  // phase cycle totals per role (debug builds only)
#define TR_DECL long long tr_acc[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tr_t0 = clock64(), tr_start = tr_t0; int tr_n = 0
#define TR_T0() (tr_t0 = clock64())
#define TR_ACC(i) do { const long long t_ = clock64(); tr_acc[i] += t_ - tr_t0; tr_t0 = t_; } while (0)
#define TR_N() (++tr_n)
#define TR_PRINT(name, xi)                                                                      \
  if (blockIdx.x == 0 || blockIdx.x == 74 || blockIdx.x == 147)                                 \
  printf("cta %d %s%d: n %d total %lld ph %lld %lld %lld %lld %lld %lld | %lld %lld | %lld %lld %lld %lld %lld\n", \
         blockIdx.x, name, (int)(xi), tr_n, clock64() - tr_start, tr_acc[0], tr_acc[1],         \
         tr_acc[2], tr_acc[3], tr_acc[4], tr_acc[5], tr_acc[6], tr_acc[7], tr_acc[8], tr_acc[9], \
         tr_acc[10], tr_acc[11], tr_acc[12])
#else
#define TR_DECL
#define TR_T0()
#define TR_ACC(i)
#define TR_N()
#define TR_PRINT(name, xi)
#endif
