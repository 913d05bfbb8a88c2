// tc_abi.h — parameter blocks shared by the host (kernels_tc.cu) and the per-plan kernels that
// are generated from tc_gate.cuh at plan registration (jit.cpp).  Plain old data only; this file
// is also spliced verbatim into the NVRTC source, so it must not include anything.
#pragma once

#define MBX_MAX_LOADS 12

// One prefetched epilogue operand: a batched or shared input row (plus column slice offset).
struct TcLoad {
  int kind;  // 0 shared, 1 batched
  int idx;   // shared / batched input index
  int off;   // column-slice offset into the input row
  int pad;
};

struct TcGateArgs {
  float* arena;
  const long long* shared_off;   // [nshared]
  const long long* batched_off;  // [b][nb]
  const long long* out_base;     // [nout] first float of each batch-contiguous output region
  const unsigned char* wpack;    // packed split-bf16 weights [unit tile][chunk][pass][128 x KC]
  int b;                         // nodes in the batch
  int NT;                        // nodes per tile (MMA N)
  int ksplit;                    // K-split ranks per tile = cluster size along z
  int stages;                    // MMA ring stages
  int nb;                        // batched inputs per node
  int npass;                     // 3: split bf16 (hi*hi + hi*lo + lo*hi), 1: bf16
  int vec16;                     // 1: every gathered row segment is 16-byte aligned
  int sep_recv;                  // unused (layout compatibility)
  int piece_kind[2], piece_idx[2], piece_off[2];
  int nloads;
  int ring_off, raw_off, recv_off, src_off, bar_off;  // dynamic shared memory layout (bytes)
  int tmem_cols;
  float* part;                   // split-K partials [tile][rank][NT][128] (ksplit > 1)
  unsigned long long* stamps;    // MBX_STAMPS builds only: [cta][8] %globaltimer phase stamps
  TcLoad loads[MBX_MAX_LOADS];
};

// One level (batch) of a persistent multi-level launch: the batch's staged offset tables.
struct TcLevel {
  const long long* shared_off;
  const long long* batched_off;
  const long long* out_base;
  int b;      // nodes in the batch
  int nt;     // node tile (MMA N) used for this level: 16, 32, 64 or MBX_LNT
  int vec16;  // 1: every gathered row segment is 16-byte aligned (bulk / 16-byte copies)
  int pad;
};

struct TcLevelsArgs {
  float* arena;
  const unsigned char* wpack;    // same packing as TcGateArgs::wpack
  const TcLevel* levels;         // [nlevels]
  int nlevels;
  int nb;
  int npass;
  int piece_kind[2], piece_idx[2], piece_off[2];
  int w_off, x_off, recv_off, bar_off;  // dynamic shared memory layout (bytes)
  int stage_off;                 // MBX_LCY > 1: row-major fp32 staging of the multicast node rows
  int tmem_cols;
  unsigned* gbar;                // grid barrier counter (monotonic across launches)
  unsigned gbar_base;            // its value when this launch starts
  float* part;                   // MBX_LXCH 1: partials [2][groups][unit tiles][S][S][MBX_LLOC][128]
  unsigned* xflags;              // MBX_LXCH 1: per (group, unit tile, rank) arrival counters, 0 at launch
  unsigned long long* stamps;    // MBX_STAMPS builds only
  TcLoad loads[MBX_MAX_LOADS];
  // MBX_FUSE_PW: a pointwise batch that consumes this (single-level) launch's rows in node order
  // runs in its tail; load pw_xt is the value just computed, the others are shared rows.
  const long long* pw_shared_off;
  const long long* pw_out_base;
  int pw_xt;
  int pw_pad;
  TcLoad pw_loads[MBX_MAX_LOADS];
};

struct SmallArgs {
  float* arena;
  const long long* shared_off;
  const long long* batched_off;
  const long long* out_base;
  int b, nb;
  int piece_kind[2], piece_idx[2], piece_off[2];
  int w_idx[4];  // shared-input index of each gate weight
  int nloads;
  TcLoad loads[MBX_MAX_LOADS];
};

struct PwArgs {
  float* arena;
  const long long* shared_off;
  const long long* batched_off;
  const long long* out_base;
  int b, E, nb, nloads;
  TcLoad loads[MBX_MAX_LOADS];
};
