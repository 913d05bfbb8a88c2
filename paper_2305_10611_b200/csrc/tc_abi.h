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
  int b;               // nodes in the batch
  int nt;              // node tile (MMA N) used for this level: 16 .. MBX_LNT
  int vec16;           // 1: every gathered row segment is 16-byte aligned (16-byte copies)
  int shadow;          // 1: every gathered row has a split-bf16 shadow (gathered MMA-ready)
  unsigned shadow_out; // bit k: write output slot k's shadow too (a later level gathers it)
  int img_slot;        // output slot whose rows are scattered into consumers' images (-1: none)
  long long img;       // byte offset (in TcLevelsArgs::img) of this level's operand image, -1: gather
  const int4* img_dst; // [b] per output row of img_slot: where its consumer's image wants it
};

struct TcLevelsArgs {
  float* arena;
  unsigned char* shadow;         // split-bf16 shadow of the arena (same float offsets, x4 bytes)
  const unsigned char* wpack;    // same packing as TcGateArgs::wpack
  const TcLevel* levels;         // [nlevels]
  int nlevels;
  int nb;
  int npass;
  int piece_kind[2], piece_idx[2], piece_off[2];
  int w_off, x_off, recv_off, bar_off;  // dynamic shared memory layout (bytes)
  int tmem_cols;
  unsigned* ready;               // per unit tile readiness counters (monotonic across launches)
  unsigned ready_base;           // their common value when this launch starts
  float* part;                   // MBX_LXCH 1: partials [2][groups][unit tiles][S][S][MBX_LLOC][128]
  unsigned* xflags;              // MBX_LXCH 1: per (group, unit tile, rank) arrival counters, 0 at launch
  unsigned long long* stamps;    // MBX_STAMPS builds only
  unsigned long long dep_mask[16]; // per K rank: unit tiles whose outputs its K slice gathers
  unsigned char* img;            // operand images (see mbx_tc_levels)
  TcLoad loads[MBX_MAX_LOADS];
};

struct SmallArgs {
  float* arena;
  const long long* shared_off;
  const long long* batched_off;
  const long long* out_base;
  const long long* out_node;  // merged launches: [b][nout] output offsets (else out_base[k] + node * U)
  unsigned long long* stamps; // MBX_SMALL_STAMPS profiling runs only: [CTA][8] globaltimer phase stamps
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
  unsigned char* shadow;  // split-bf16 shadow of the arena (16-byte variants only)
  unsigned shadow_out;    // bit k: write output slot k's shadow too
  int img_slot;           // output slot scattered into consumers' operand images (-1: none)
  unsigned char* img;     // operand images
  const int4* img_dst;    // [b] per output row of img_slot (see mbx_tc_levels)
  int b, E, nb, nloads;
  TcLoad loads[MBX_MAX_LOADS];
};
