// Internal interfaces of the batched planner (plan.cu) and the rectangle
// validator (validate.cu).
#pragma once
#include "batch.cuh"

namespace stw {

// sort by the composite key (hi, lo) of widths (hibits, lobits); perm[k] =
// index of the k-th smallest. hi/lo are consumed (overwritten).
void sort_perm2(Ctx &ctx, Arena &ar, uint64_t *hi, int hibits, uint64_t *lo, int lobits, uint32_t *perm,
                int64_t n);

// Static rectangles of a batch of decision sets, set s = [off[s], off[s+1]),
// each set listed in its sweep order ((t_s, id) order). ts/te/rank are per
// rectangle; addr/size per (candidate, rectangle) with stride `stride`.
struct RectSets {
  int32_t S;            // number of sets (traces)
  int64_t n;            // rectangles in all sets
  const int64_t *off;   // [S+1] device
  const int32_t *ts, *te;  // [n] in sweep order
  const int64_t *size;     // [n]
  int32_t n_cand;
  const int64_t *addr;     // [n_cand * n] (candidate-major)
};

// K7 for the planner self-check: per (set, candidate) the number of pairs the
// reference sweep (planner.py:476-505) would report and the sweep position of
// the first reporting decision (INT_MAX if none). Outputs are device arrays of
// S*n_cand entries, unit index = set*n_cand + cand.
// Addresses and sizes are expected to be multiples of 2^shift (the alignment);
// units that are not fall back to the exact tiled reporter.
void validate_sets(Ctx &ctx, Arena &ar, const RectSets &rs, long long *d_count, int *d_first, int shift);

// Fast exact validity test (no report) of every (set, candidate); returns the
// number of units that need the exact reporter (0 = every unit is valid), -1
// on a CUDA error.
int overlap_flags(Ctx &ctx, Arena &ar, const RectSets &rs, int shift);
// the same test without the host round trip: returns the device counter
// order (optional, device): the sets in launch order (largest first evens out the
// tail of the one-warp-per-unit sweep)
int *overlap_launch(Ctx &ctx, Arena &ar, const RectSets &rs, int shift, const int32_t *order = nullptr);
// the exact reporter for every unit (fills d_count / d_first)
void validate_exact(Ctx &ctx, Arena &ar, const RectSets &rs, long long *d_count, int *d_first);

// Host-side re-derivation of the first reported pair (a, b) of a decision set
// whose first reporting decision is at sweep position `first` (device data).
void first_pair(Ctx &ctx, const RectSets &rs, int set, int cand, int first, int *pa, int *pb);

// Register-resident sequential replay (replay_reg.cu) of one trace: inputs in
// op order (operm: op 2e = alloc of event e, 2e+1 = its free; apos[e] = op
// index of e's alloc), routes / planned addresses from the queue matching.
// Requires unique ids. Returns 0 done (hout[4..10] = metrics, the log written
// when asked), 1 outside its preconditions (the caller runs k_replay), 2 a
// replay error (hout[1] code, hout[2] id, hout[3] address).
struct RegIn {
  int64_t n;
  const uint32_t *operm;
  const int32_t *apos;
  const int64_t *id, *size;
  const int32_t *ts, *te;
  const uint8_t *dyn;
  const int8_t *route0;
  const int64_t *paddr;
  const int32_t *key;
  const int64_t *sp_off, *sp_lo, *sp_hi;
  int64_t nsp;
  int reuse, baseline;
  long long pool;
  // simulate only: planned static allocations off the sequential chain (see
  // offchain_check): full op -> kept op index, and the kept op count; nullptr:
  // every op is replayed
  const uint32_t *ridx;
  int64_t nkept;
};
int replay_reg(Ctx &ctx, Arena &ar, RegIn &in, long long *hout, stw_log *log);
// true when the planned static allocations of a simulate call can leave the
// sequential chain; then in.ridx / in.nkept are set
bool offchain_check(Ctx &ctx, Arena &ar, RegIn &in, int64_t nkeys);

}  // namespace stw
