// libhps_gpu.so — the B200-native HBM-PS tier behind the C ABI of
// include/hps_gpu.h. One handle per GPU (rank g of G = nodes * devices).
//
// Per batch (hps_train_batch), all on the handle's stream:
//   batch_count  -> one D2H of the per-mini-batch occurrence counts
//   working set  -> radix sort + unique of the rank's owned keys (a1, a2)
//   build        -> capacity, clear, ordered-probing insert, row fill with
//                   carry-over / store staging (a3, a4)
//   J x mini-batch:
//     shard gather, radix sort (key, occurrence), unique -> inverse index
//     and CSR segments (a5); [G>1: stable owner partition, count
//     all-gather, key all-to-all]; owner probe+gather (a6) [G>1: row
//     all-to-all]; fwd/bwd (a7, a8); dense-grad reduce; sparse
//     segment-reduce + sgd_delta (a8, a9) [G>1: delta all-to-all (a10)];
//     canonical owner apply (a11); dense sync + update (a12)
//   write-back   -> rows to the value store (a13)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "hps_gpu.h"
#include "model.cuh"
#include "p2p.cuh"
#include "sort.cuh"
#include "table.cuh"
#include "group.cuh"
#include "mlp.cuh"
#include "tier_internal.h"

namespace hpsgpu {

thread_local std::string t_err;
void set_error_message(const std::string& m) { t_err = m; }
const char* error_message() { return t_err.c_str(); }

// ------------------------------------------------------------- NCCL ----
// Loaded with dlopen so the library (and the CPU test suite) does not need
// NCCL unless a tier spans more than one GPU; inside a torch process this
// resolves to the NCCL torch already loaded.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t,
                            ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      a.why = "cannot dlopen libnccl.so.2";
      return a;
    }
#define HPS_SYM(field, name)                                            \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(lib, name));      \
  if (!a.field) {                                                       \
    a.why = std::string("missing NCCL symbol ") + name;                 \
    return a;                                                           \
  }
    HPS_SYM(GetUniqueId, "ncclGetUniqueId");
    HPS_SYM(CommInitRank, "ncclCommInitRank");
    HPS_SYM(CommDestroy, "ncclCommDestroy");
    HPS_SYM(GroupStart, "ncclGroupStart");
    HPS_SYM(GroupEnd, "ncclGroupEnd");
    HPS_SYM(Send, "ncclSend");
    HPS_SYM(Recv, "ncclRecv");
    HPS_SYM(AllGather, "ncclAllGather");
    HPS_SYM(AllReduce, "ncclAllReduce");
    HPS_SYM(GetErrorString, "ncclGetErrorString");
#undef HPS_SYM
    a.ok = true;
    return a;
  }();
  return api;
}

// --------------------------------------------------------- the tier ----

// tables: current, previous (carry-over), two older ones whose rows stand in
// for the store (store proxies, copied by the body), and one more so the
// table a body reads as its oldest proxy is recycled two builds later
constexpr int kTables = 5;
constexpr int kSlots = 5;   // staging slots (rotating with the tables: one graph per slot per shape)
constexpr int kMaxInflight = 4;  // batches in flight

struct Scalars {
  std::uint64_t n_ws;          // working-set size of the current build
  std::uint64_t cap[kTables];      // capacity of each table
  std::uint64_t nws_tab[kTables];  // occupancy of each table
  unsigned long long carried_tab[kTables];  // rows carried over when the table was built
  unsigned long long stored_tab[kTables];   // rows read from the value store for it
  std::uint64_t U;             // unique keys of the current mini-batch / pull
  std::uint64_t counts[kSlots][66]; // batch_count per staging slot: per-mb occurrences, owned keys
  double loss;
  unsigned long long pulled;   // sum over mini-batches of unique keys pulled
  unsigned long long carried;  // rows filled from the previous table
  unsigned long long n_long;   // medium CSR segments queued this mini-batch
  unsigned long long n_big;    // big segments (split over CTAs)
  unsigned long long n_items;  // their (key, chunk) work items
  int err_any;                 // error code max-reduced over ranks
  unsigned long long epoch;    // P2P exchange round (parity selects the windows)
  std::uint32_t pad0, pad1;
  std::int64_t total_unused;   // host side: offsets[B] of a device batch
  unsigned long long gn[4];      // grouping (prep lane): n_long, n_dup, n_huge
  unsigned long long wb_n[kTables];  // rows on each table's write-back list
  unsigned long long wb_total;       // rows written to the store (cumulative)
  unsigned long long Ug[kTables][64];  // unique keys per (table, mini-batch), grouped path
  std::uint64_t rq_capv;               // request-table capacity (G > 1)
  unsigned spec_fail, redo;            // speculative table build (prep)
  unsigned long long fallbacks;  // certified sums that needed the exact chain
  unsigned long long served;     // keys this rank served as owner (G > 1)
  unsigned long long big_keys;   // segments on the chunked path (this batch)
  unsigned long long max_chunks; // most chunks of one of them
  unsigned long long big_occ;    // their occurrences
  unsigned long long mid_keys;   // segments on the exact warp-chain path (this batch)
  unsigned long long n_mid;      // this mini-batch's medium segments
  unsigned long long Ux[2];      // fused exchange: unique keys of mini-batch j, by j & 1
  unsigned long long xclear[2];  // (scratch for owner_rank_kernel's clear words)
  unsigned long long xscratch[4];  // (scratch: the prep's owner-rank pass opens no round)
  DevError err;                 // the body's and the parity API's error word
  // per-batch error words of the pipelined stages: the stage's
  // key-range check (by staging slot) and the prep's build (by table), so an
  // in-flight batch's error is never read or cleared by another batch
  DevError serr[kSlots];
  DevError perr[kTables];
};

struct BatchShape {
  std::uint64_t B = 0;
  std::uint64_t own_bound = 0, batch_bound = 0;
  std::uint64_t mb_bound[64] = {};
};

// Which buffers one in-flight batch uses (hps_submit_batch).
struct BatchPlan {
  std::uint64_t id = 0;  // submission index
  std::uint64_t B = 0;
  int sp = 0;         // staging slot (double-buffered batch + counts)
  int tb = 0;         // its table
  int tp = -1;        // previous table (carry-over), -1 = none
  int tq = -1;        // table two builds back, usable as a store proxy, -1 = none
  int tq2 = -1;       // three builds back, likewise
  std::int64_t step = 0;
  std::uint64_t occ_total = 0;
  int skip_mb = -1;
  bool grouped = false;  // slot grouping (prep lane, and the body's side branch)
  int prep_mbs = 0;      // mini-batches grouped by the prep
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  std::uint64_t last_use = 0;  // LRU eviction
  std::uint64_t launches = 0;
  std::uint64_t epochs = 0;  // exchange rounds the body opens (host mirror)
  std::vector<int> ev_phase, ev_lane;
};

// A stream with its own sort / scan scratch and look-back state, so the
// build of batch b+1 (prep lane) and the body of batch b (main lane) can run
// concurrently.
struct LaneDev {
  std::uint64_t total;      // scratch total of a tile scan
  std::uint32_t context;    // look-back context counter (sort.cuh)
  std::uint32_t pad;
};
struct Lane {
  cudaStream_t st = nullptr;
  std::uint64_t *kA = nullptr, *kB = nullptr;
  std::uint32_t *vA = nullptr, *vB = nullptr;
  std::uint32_t* ghist = nullptr;          // [kMaxPasses][256] digit bases
  std::uint64_t* status = nullptr;         // look-back status words
  unsigned long long* ticket = nullptr;    // look-back tile tickets
  LaneDev* d = nullptr;
  std::uint64_t tickets = 0;               // tickets handed out in this context
  std::uint32_t lb_local = 0;              // launches in this context
  std::uint64_t lb_contexts = 0;           // contexts opened (host mirror)
  std::uint64_t status_words = 0;
};

// The temporaries of one grouping context: the prep's (lane 2) and the
// body's (lanes 3 and 4: the body's later mini-batches alternate between
// them, so two groupings run side by side).
constexpr int kGroupLanes = 4;
struct GroupState {
  std::uint32_t* gcnt = nullptr;       // [gslots] per-slot occurrence counters (kept zero)
  std::uint32_t* slot_uid = nullptr;   // [gslots]
  std::uint32_t* part_slot = nullptr;  // [kGroupParts][part_cap] claimed slots
  std::uint32_t* part_n = nullptr;     // [kGroupParts * kGroupPartStride] claim counters
  std::uint32_t* part_base = nullptr;  // [kGroupParts]
  std::uint32_t *g_long = nullptr, *g_huge = nullptr, *g_dup = nullptr;  // segment lists
  unsigned long long* gn = nullptr;    // [4] n_long, n_dup, n_huge
  cudaEvent_t join = nullptr, ctx = nullptr;
};

// Per-batch results read back at hps_wait_batch (pinned).
struct BatchOut {
  double loss;
  unsigned long long pulled;
  unsigned long long fallbacks, served, big_keys, max_chunks, big_occ, mid_keys;
  unsigned long long carried, stored;
  std::uint64_t n_ws, cap;
  DevError err, err_stage, err_prep;
};

// A batch's readback (loss, counters, error words) in ONE launch after its
// body: one thread copies the fields into the slot's pinned BatchOut (mapped,
// UVA) — nine small D2H copies serialised the body stream by ~30 us.
__global__ void batch_out_kernel(const Scalars* __restrict__ d, int tb, int sp,
                                 BatchOut* __restrict__ o) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  o->loss = d->loss;
  o->pulled = d->pulled;
  o->fallbacks = d->fallbacks;
  o->served = d->served;
  o->big_keys = d->big_keys;
  o->max_chunks = d->max_chunks;
  o->big_occ = d->big_occ;
  o->mid_keys = d->mid_keys;
  o->carried = d->carried_tab[tb];
  o->stored = d->stored_tab[tb];
  o->n_ws = d->nws_tab[tb];
  o->cap = d->cap[tb];
  o->err = d->err;
  o->err_stage = d->serr[sp];
  o->err_prep = d->perr[tb];
}

// Zeroes up to kZeroRegions small device regions (u32 words) in ONE launch:
// inside the captured graphs a memset node breaks the programmatic-launch
// chain and costs ~5 us of dependency latency each; the CUPTI timeline
// showed chains of 2-5 of them at the head of every mini-batch's reduce,
// grouping and build.
constexpr int kZeroRegions = 6;
struct ZeroList {
  std::uint32_t* p[kZeroRegions];
  std::uint32_t n[kZeroRegions];  // words
};
__global__ void zero_kernel(ZeroList z) {
  pdl_wait();
#pragma unroll
  for (int r = 0; r < kZeroRegions; ++r)
    for (std::uint32_t i = threadIdx.x; i < z.n[r]; i += blockDim.x) z.p[r][i] = 0u;
}

// Copy-back of a mirrored store at G > 1: the rows this rank owns (key % G
// == g) in the dirty pages, straight into the mapped host array (the ranks
// may share it; each writes only its own rows, as the per-batch write-back
// does).
__global__ void mirror_owned_copyback_kernel(const float4* __restrict__ mirror,
                                             float4* __restrict__ host,
                                             const std::uint8_t* __restrict__ pages,
                                             std::uint64_t num_keys, int rw4, int G, int g) {
  pdl_wait();
  const std::uint64_t total = num_keys * std::uint64_t(rw4);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t key = t / std::uint64_t(rw4);
    if (key % std::uint64_t(G) != std::uint64_t(g) || !pages[key >> 10]) continue;
    host[t] = mirror[t];
  }
}

// One sender's pushed (keys, deltas) awaiting hps_drain: a range of the
// pending arena (Tier::pend_*), which grows by doubling and is reused.
struct PendingChunk {
  int src;
  std::uint64_t n;
  std::uint64_t at;  // first entry in the arena
};

struct Tier {
  hps_config cfg{};
  int N = 1, D = 1, G = 1, g = 0, E = 1, J = 1;
  int RW = 1;   // floats per table / store row: E, or 2E with the Adagrad state
  Optim opt{};  // the sparse optimizer the owners apply (common.cuh)
  ModelDims md{};
  cudaStream_t st = nullptr;            // == lane[0].st: bodies and the parity API
  cudaStream_t st2 = nullptr;           // side stream: dense-grad overlaps sparse reduce
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaStream_t st3 = nullptr;           // side stream: the big-segment path (classify, plan,
  cudaEvent_t fork3 = nullptr, join3 = nullptr;  // fused reduce) beside fwd/bwd + short path
  cudaStream_t st4 = nullptr;           // side stream: the medium segments (sparse_mid_kernel)
  cudaEvent_t fork4 = nullptr, join4 = nullptr;
  int short_dpt = 0;                    // sparse_short dims per thread (HPS_SHORT_DPT; 0 = auto)
  std::uint32_t mid_max = 512;          // medium segments: short_max < length <= mid_max
  std::uint32_t short_max = 32;         // short segments (thread chains): length <= short_max
  int prep_group_lanes = 2;  // lanes grouping the prep's mini-batches (HPS_PREP_GROUP_LANES)
  int body_group_lanes = 2;  // lanes grouping the body's later mini-batches (HPS_BODY_GROUP_LANES)
  bool fb_fixed = true;  // fwd/bwd with the {8, 16, 1} stack at compile time (HPS_FB_FIXED=0: generic)
  unsigned short_grid = 8 * kSMs;  // block cap of sparse_short_kernel (HPS_SHORT_GRID; 0: kSMs * 32)
  int prog_edges = 1;  // programmatic graph edges: 1 fwd/bwd -> side reduces, 2 all kernel->kernel,
                       // 3 also side reduces -> dense update, 4 every kernel edge into a side
                       // reduce (HPS_PROG_EDGES)
  bool prep_lag1 = false;  // the build waits for the previous body's carry (HPS_PREP_LAG=1)
  bool dg_main = false;  // dense gradient on the body stream, short keys on st2 (HPS_DG_MAIN)
  bool tail_prio = false;  // st3/st4 above st/st2 (HPS_TAIL_PRIO=1; measured no gain on c2)
  bool group_fused = true;  // segment ordering in one launch (HPS_GROUP_FUSED=0: four)
  bool group_prio = false;  // the body's own grouping lane at body priority (HPS_GROUP_PRIO=1)
  unsigned prep_grid = 4 * kSMs;  // HPS_PREP_GRID: block cap of the prep-side kernels (0: none)
  bool mid_cert = true;  // medium segments certified (HPS_MID_CERT=0: exact warp chains)
  bool dg_fused = true;  // dense gradient in one launch (HPS_DG_FUSED=0: four launches)
  bool fb_tile = true;  // fwd/bwd embed_sum through shared-memory row tiles (HPS_FB_TILE=0: off)
                                        // (HPS_MID_SEG; kLongSeg disables the path)
  Lane lane[2 + kGroupLanes];           // 0: main (body), 1: prep (build of the next batch),
                                        // 2..: the next batch's mini-batch groupings
  GroupState gs[kGroupLanes];           // the prep's groupings first, then the body's
  int prep_mbs = 0;                     // mini-batches the prep groups (HPS_PREP_GROUP;
                                        // 0 = auto); the body groups the rest, each
                                        // beside the previous mini-batch's compute
  cudaEvent_t gmb_done[64] = {};        // body grouping: mini-batch j ready
  cudaEvent_t b_fork = nullptr;
  cudaEvent_t g_fork = nullptr;
  Lane* L = &lane[0];                   // the lane launch() enqueues on
  // The batch pipeline (the reference's 4-stage pipeline, pipeline.hpp:230-
  // 500, as streams): stage (H2D + counts, st_stage) -> prep (working set,
  // table build, store prefetch; lane 1) -> body (carry + J mini-batches;
  // lane 0) -> write-back (st_wb, the collect stage, pipeline.hpp:462-474).
  // Batch b+1 is staged and prepared while batch b trains; b's write-back
  // overlaps b+1.
  cudaStream_t st_stage = nullptr, st_wb = nullptr;
  cudaStream_t st_pf = nullptr;         // prep's store gather, forked beside the grouping
  cudaEvent_t pf_fork = nullptr, pf_join = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_prep = nullptr;
  cudaEvent_t ev_body_tab[kTables] = {}, ev_body_sp[kSlots] = {}, ev_wb[kTables] = {};
  cudaEvent_t ev_carry_sp[kSlots] = {};  // a body's resident-table copies are done
  cudaEvent_t ev_wbt[kTables][2] = {};  // write-back timing pairs
  bool body_pending[kTables] = {}, sp_pending[kSlots] = {}, wb_pending[kTables] = {},
       wb_timed[kTables] = {};
  bool tab_wb[kTables] = {};            // a train table of the current store (its rows
                                        // reach the store on eviction or flush)
  bool tab_flushed[kTables] = {};       // ... and they are there already
  std::uint64_t tab_age[kTables] = {};  // build order
  std::uint64_t builds = 0;
  std::uint64_t rows_read = 0;          // store rows read (completed batches, cumulative)
  std::deque<BatchPlan> inflight;       // submitted, not yet completed (<= kSlots)
  struct Done {
    std::uint64_t id;
    hps_status st;
    std::string msg;
    hps_batch_stats stats;
  };
  std::deque<Done> done;                // completed, not yet returned
  std::uint64_t submitted = 0;
  ncclComm_t comm = nullptr;
  std::uint64_t Bmax = 0, Omax = 0, Wmax = 0, capmax = 0, nmb_max = 0;
  int sort_bits = 64;
  std::uint64_t launches = 0;
  std::int64_t step = 0;  // batches trained (global mini-batch = step*J + j)

  Scalars* dsc = nullptr;  // device
  Scalars* hsc = nullptr;  // pinned host mirror

  // tables (triple-buffered: current, previous for carry-over, and the one
  // before, whose rows stand in for the store while its write-back drains)
  std::uint64_t* tkeys[kTables] = {};
  float* tvals[kTables] = {};
  int cur = -1, prev = -1, prev2 = -1;
  int hist[kTables] = {-1, -1, -1, -1, -1};  // table of the k-th most recent build

  // working set
  std::uint64_t* ws = nullptr;       // sorted keys of the current table (when ws_sorted)
  std::uint32_t* ws_idx = nullptr;   // (ws / ws_idx point into wsb / wsib of the table)
  std::uint64_t* wsb[kTables] = {};
  std::uint32_t* wsib[kTables] = {};
  std::uint32_t* csrc[kTables] = {};  // carry source slot per working-set entry
  bool ws_sorted = true;

  // batch staging (double-buffered)
  std::int64_t* b_off[kSlots] = {};
  std::uint64_t* b_keys[kSlots] = {};
  std::uint8_t* b_lab[kSlots] = {};
  BatchOut* hout = nullptr;          // pinned, [kSlots] by staging slot

  // mini-batch / pull buffers (sized Omax)
  std::uint32_t *occ_off = nullptr, *ex_of = nullptr, *inv = nullptr,
                *seg = nullptr, *uidv = nullptr, *pos = nullptr,
                *slots = nullptr,
                *exs = nullptr,
                *big_list = nullptr, *chunk_off = nullptr, *mid_list = nullptr,
                *orank = nullptr,
                *key_done = nullptr;
  ChunkSum* chunk_tot = nullptr;
  std::uint32_t *item_key = nullptr, *item_chunk = nullptr;  // item -> (big key, chunk)
  unsigned long long* fuse_ticket = nullptr;
  std::uint64_t fuse_items = 0;
  std::uint64_t* otot = nullptr;
  std::uint64_t* ukeys = nullptr;
  // fused exchange (G > 1, grouped; HPS_XFUSE=0: the four-phase exchange):
  // unique keys, owner ranks and per-owner counts of mini-batch j, by j & 1
  bool xfuse = true;
  std::uint64_t* xukeys[2] = {};
  std::uint32_t* xorank[2] = {};
  std::uint64_t* xotot[2] = {};
  // ... computed by the prep's grouping instead (per table, mini-batch j at
  // its grouping region; HPS_XPREP=0: in the body, x_keys)
  bool xprep = true;
  std::uint64_t* pxukeys[kTables] = {};
  std::uint32_t* pxorank[kTables] = {};
  std::uint64_t* pxotot[kTables] = {};   // [64][kMaxRanks]
  float *rows = nullptr, *deltas = nullptr, *hstage = nullptr, *staged = nullptr;
  std::uint64_t staged_cap = 0;  // floats

  // model
  double *H = nullptr, *DL = nullptr, *DX = nullptr, *dpart = nullptr;
  // wide MLP path (mlp.cuh; a hidden layer wider than kMaxHidden, or
  // HPS_WIDE=1): per-shard activations and deltas (f32, [nshard][width]),
  // split-K partials of the weight gradients
  bool wide = false;
  bool gemm_split3 = true;   // 3xTF32 (HPS_TF32_1X=1: plain TF32)
  std::uint64_t nshard = 0;  // examples of a mini-batch shard, at most
  float* wX = nullptr;
  float* wH[kMaxLayers] = {};
  float* wdZ[kMaxLayers] = {};
  float* wdz = nullptr;
  float* wP = nullptr;
  std::uint64_t wP_cap = 0;
  double *dg_off = nullptr, *dg_tot = nullptr;  // dense-grad slice offsets, totals
  unsigned* dg_sync = nullptr;  // dense_grad_fused_kernel: per weight group, CTAs counted
  float *dense = nullptr, *dgrad = nullptr;

  // value store (MEM-PS stand-in)
  float* store = nullptr;
  std::uint64_t store_keys = 0;
  bool store_on_host = false;
  // host value store mirrored in HBM (HPS_STORE_MIRROR_GB, default 2: a
  // store that fits is copied to the device once at attach, trained there,
  // and its dirty pages copied back whenever the host observes it, i.e. at
  // every quiesce after a write-back; bigger stores, whose copy-back would
  // cost more than a short run's per-batch staging, stay on the host)
  float* mirror = nullptr;
  float* mirror_host = nullptr;
  std::uint64_t mirror_bytes = 0;
  bool mirror_dirty = false;
  double mirror_gb = 2.0;
  std::uint8_t* mirror_pages = nullptr;  // dirty flag per 2^kMirrorPageShift-row page
  std::uint64_t mirror_h2d = 0, mirror_d2h = 0;  // bytes the mirror moved over PCIe
  std::vector<std::uint8_t> mirror_hpages;
  float* mirror_hmapped = nullptr;  // G > 1: the host array's device mapping (owned-row copy-back)
  bool mirror_registered = false;
  // zero-copy kernels on a host store run on a few SMs only: a PCIe access
  // stalls the memory pipeline of the SM issuing it for everyone on that SM
  unsigned pf_ctas = 8, wb_ctas = 4;
  bool hash_dedup = true;                // group.cuh at G == 1 (HPS_DEDUP=sort: radix sort)
  // slot grouping outputs, per table (prep of b+1 writes while body b reads):
  // occurrence -> slot (batch key index), and per mini-batch region (at the
  // sum of the earlier mini-batches' shape bounds) segments, example ids,
  // uid -> slot; uid counts in Scalars::Ug
  std::uint32_t* g_occslot[kTables] = {};
  std::uint32_t* g_inv[kTables] = {};      // G > 1: occurrence -> uid (rows come in uid order)
  std::uint64_t* rq_keys[kTables] = {};    // G > 1: request table, the rank's shard keys
  std::uint64_t rq_cap = 0;
  std::uint64_t gslots = 0;                 // entries of gcnt / slot_uid
  std::uint32_t* g_segb[kTables] = {};
  std::uint32_t* g_exsb[kTables] = {};
  std::uint32_t* g_uidb[kTables] = {};
  std::uint64_t g_pool = 0;              // region pool size (elements)
  // prep-only temporaries of the grouping
  // occurrence-indexed temporaries, per table: a prep groups batch b+1 while
  // the body of batch b groups its own later mini-batches
  std::uint32_t* g_tick[kTables] = {};
  std::uint32_t* g_segocc[kTables] = {};
  std::uint32_t* g_exof[kTables] = {};

  std::uint64_t part_cap = 0;
  // HPS_TRACE=1: timed events at the pipeline's stage boundaries, printed
  // per batch to stderr at completion (diagnostics)
  bool trace = false;
  bool priorities = true;
  bool big_side = true;
  bool fold_wait = true;  // the exchange waits inside the consuming kernel (HPS_FOLD_WAIT=0: own launch)
  int ws_sort = -1;  // prep sorts the working set by key: 1/0 (HPS_WS_SORT), -1 = for a host store                 // big-segment path on st3 (HPS_BIG_SIDE=0: on st)
  int zc_threads = 1024;  // CTA size of the zero-copy kernels
  cudaEvent_t tr_base = nullptr;
  cudaEvent_t tr[kSlots][6] = {};   // by staging slot: stage0 stage1 prep0 prep1 body0 body1
  cudaEvent_t trw[4][2] = {};  // write-back start/end by batch id % 4
  cudaEvent_t trg[kSlots][2] = {};  // store gather start/end by staging slot
  std::uint64_t* need_key[kTables] = {};   // store rows of each table's build
  std::uint32_t* need_slot[kTables] = {};
  std::uint64_t* wb_key[kTables] = {};     // each table's write-back list
  std::uint32_t* wb_slot[kTables] = {};
  bool store_registered = false;
  float* store_host = nullptr;
  // MEM-PS staging through host threads + DMA (HPS_STAGE=dma; zero-copy SM
  // gathers are the default, measured faster here): the store rows a build needs are gathered
  // by host threads into pinned staging and copied with one cudaMemcpyAsync;
  // the evicted rows are compacted on the device, copied back with one
  // cudaMemcpyAsync and scattered into the store by host threads. Zero-copy
  // SM gathers of random 64-byte host rows reach ~11 GB/s on c5; 16 host
  // threads gather at 22-30 GB/s and the DMA runs at ~55 GB/s (round 1,
  // tools/pcie_probe.cu).
  int stage_mode = -1;  // HPS_STAGE: 1 dma, 0 zero-copy, -1 auto
  bool dma = false;
  float* store_hptr = nullptr;           // the host store (pinned or pageable)
  struct DmaJob {
    const std::uint64_t* cnt;            // pinned: rows in this transfer
    const std::uint64_t* keys;           // pinned: their keys
    float* rows;                         // pinned staging rows
    float* store;
    int RW;
    int threads;
    bool scatter;                        // false: store -> rows, true: rows -> store
  };
  DmaJob gjob{}, wjob{};
  std::uint64_t *g_hcnt = nullptr, *g_hkeys = nullptr, *w_hcnt = nullptr, *w_hkeys = nullptr;
  float *g_hrows = nullptr, *w_hrows = nullptr;  // pinned staging
  float *g_drows = nullptr, *w_drows = nullptr;  // device staging
  std::vector<void*> pinned;

  std::vector<PendingChunk> pending;
  std::uint64_t* pend_keys = nullptr;  // the pending arena (hps_push -> hps_drain)
  float* pend_deltas = nullptr;
  std::uint64_t pend_cap = 0, pend_used = 0;

  // in-kernel NVLink all-to-all (G > 1): this rank's exported window and the
  // peers' windows (p2p.cuh)
  // Windows are double-buffered by round parity (epoch & 1) so a fast rank
  // never overwrites a region a slower peer is still reading.
  // The round counter lives in device memory (Scalars::epoch); kernels pick
  // the parity themselves, so captured graphs stay valid across replays.
  P2PCtx ctx{};
  std::uint64_t slot = 0;            // per-source region capacity (keys)
  std::uint64_t* w_keys_p[2] = {};   // this rank's windows, per parity: [G][slot]
  std::uint64_t* w_hdr_p[2] = {};    // [G][2]
  float* w_deltas_p[2] = {};         // [G][slot][E]
  float* w_dense_p[2] = {};          // [G][nw]
  std::uint64_t* w_flags = nullptr;  // [G][kPhases] (monotonic epochs)
  std::uint32_t* w_rslots = nullptr; // [G][slot] cached owner slots (local)
  unsigned* done_ctr = nullptr;
  std::uint64_t p2p_epoch = 0;
  void* win_base = nullptr;
  std::vector<void*> ipc_opened;

  // timing: events recorded at phase boundaries on the lanes' streams
  bool timing = false;
  std::vector<cudaEvent_t> evpool;
  std::vector<int> ev_phase, ev_lane;  // lane: 0 main, 1 prep, 2 stage
  double acc_ms[HPS_TIMING_SLOTS] = {0};

  std::vector<void*> allocs;

  // captured per-batch graphs (hps_train_batch), keyed by the batch shape
  bool use_graphs = true;
  std::map<std::vector<std::uint64_t>, GraphEntry> graphs;
  std::uint64_t graph_clock = 0;     // LRU clock of the graph cache
  std::vector<cudaGraphExec_t> retired;  // evicted graphs, destroyed once nothing is in flight
  std::uint64_t graph_captures = 0;  // captures so far (diagnostics, bench)
};

// ----------------------------------------------------------- helpers ----

#define HPS_CUDA(call)                                                      \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      return set_error(HPS_ERR_CUDA, "cuda: %s at %s:%d", cudaGetErrorString(e_), \
                       __FILE__, __LINE__);                                 \
  } while (0)

#define HPS_TRY(expr)                  \
  do {                                 \
    hps_status s_ = (expr);            \
    if (s_ != HPS_OK) return s_;       \
  } while (0)

#define HPS_NCCL(call)                                                     \
  do {                                                                     \
    ncclResult_t r_ = (call);                                              \
    if (r_ != ncclSuccess)                                                 \
      return set_error(HPS_ERR_NCCL, "nccl: %s at %s:%d",                  \
                       nccl().GetErrorString(r_), __FILE__, __LINE__);     \
  } while (0)

template <class T>
static hps_status dalloc(Tier* t, T** p, std::uint64_t count) {
  void* q = nullptr;
  const std::uint64_t bytes = std::max<std::uint64_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess)
    return set_error(HPS_ERR_CUDA, "cuda: cudaMalloc(%llu B): %s",
                     (unsigned long long)bytes, cudaGetErrorString(e));
  t->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return HPS_OK;
}

static unsigned grid_for(std::uint64_t work, int threads = 256,
                         unsigned cap = kSMs * 16) {
  const std::uint64_t b = (work + threads - 1) / threads;
  return unsigned(std::max<std::uint64_t>(1, std::min<std::uint64_t>(b, cap)));
}

// Grid of a prep-side (off the critical path) grid-stride kernel: capped at
// Tier::prep_grid blocks (HPS_PREP_GRID; 0 = uncapped) so that the batch
// build never fills every SM while the body's kernels wait for slots.
struct Tier;
static unsigned prep_grid_of(const Tier* t, unsigned g);

bool debug_sync_enabled();

// HPS_DEBUG_SYNC=1 (diagnostics, graphs must be off): synchronise after every
// launch and name the kernel that failed.
template <class K>
static void debug_sync(K* k, cudaStream_t s) {
  if (!debug_sync_enabled()) return;
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    const char* name = "?";
    cudaFuncGetName(&name, reinterpret_cast<const void*>(k));
    std::fprintf(stderr, "[hps debug] kernel %s: %s\n", name, cudaGetErrorString(e));
  }
}

bool pdl_enabled();

// Every launch allows programmatic dependent launch (see pdl_wait): the
// kernel's blocks may start as the predecessor's last ones drain.
template <class... KArgs, class... Args>
static void launch_on(Tier* t, cudaStream_t s, void (*k)(KArgs...), dim3 grid, dim3 block,
                      size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
  ++t->launches;
  debug_sync(k, s);
}

template <class... KArgs, class... Args>
static void launch(Tier* t, void (*k)(KArgs...), dim3 grid, dim3 block,
                   size_t smem, Args&&... args) {
  launch_on(t, t->L->st, k, grid, block, smem, std::forward<Args>(args)...);
}


// Maps the device error word to the reference's hps::Error texts. With
// collective = true (calls every rank makes in lockstep) the error code is
// max-reduced over ranks first, so an owner-side failure (e.g. a missing key
// requested by a peer) makes every rank raise instead of diverging.
static hps_status device_error_status(Tier* t, const DevError& e, const char* missing_ctx);

static hps_status check_device_error(Tier* t, const char* missing_ctx,
                                     bool collective = false, cudaStream_t s = nullptr,
                                     DevError* slot = nullptr) {
  if (!s) s = t->st;
  if (!slot) slot = &t->dsc->err;
  if (collective && t->G > 1) {
    HPS_CUDA(cudaMemcpyAsync(&t->dsc->err_any, &slot->code, sizeof(int),
                             cudaMemcpyDeviceToDevice, s));
    ncclResult_t r = nccl().AllReduce(&t->dsc->err_any, &t->dsc->err_any, 1, ncclInt32, ncclMax,
                                      t->comm, s);
    if (r != ncclSuccess)
      return set_error(HPS_ERR_NCCL, "nccl: %s", nccl().GetErrorString(r));
    HPS_CUDA(cudaMemcpyAsync(&t->hsc->err_any, &t->dsc->err_any, sizeof(int),
                             cudaMemcpyDeviceToHost, s));
  }
  HPS_CUDA(cudaMemcpyAsync(&t->hsc->err, slot, sizeof(DevError), cudaMemcpyDeviceToHost, s));
  HPS_CUDA(cudaStreamSynchronize(s));
  const DevError e = t->hsc->err;
  if (e.code == 0 && collective && t->G > 1 && t->hsc->err_any != 0)
    return set_error(hps_status(t->hsc->err_any),
                     "hbm: a peer rank failed this collective (status %d)", t->hsc->err_any);
  if (e.code == 0) return HPS_OK;
  HPS_CUDA(cudaMemsetAsync(slot, 0, sizeof(DevError), s));
  return device_error_status(t, e, missing_ctx);
}

static hps_status device_error_status(Tier* t, const DevError& e, const char* missing_ctx) {
  if (e.code == 0) return HPS_OK;
  const unsigned long long k = e.key;
  switch (e.code) {
    case HPS_ERR_MISSING_KEY:
      return set_error(HPS_ERR_MISSING_KEY, "%s%llu", missing_ctx, k);
    case HPS_ERR_DUPLICATE:
      return set_error(HPS_ERR_DUPLICATE,
                       "device table: duplicate insert of key %llu", k);
    case HPS_ERR_OVERFLOW:
      return set_error(HPS_ERR_OVERFLOW,
                       "device table: capacity overflow (sizing bug)");
    case HPS_ERR_NONFINITE:
      return set_error(HPS_ERR_NONFINITE, "model: non-finite value");
    case HPS_ERR_KEY_RANGE:
      return set_error(HPS_ERR_KEY_RANGE,
                       "ingest: feature key %llu out of range for dims=%llu",
                       k, (unsigned long long)t->cfg.key_space);
    case HPS_ERR_ARG:
      return set_error(HPS_ERR_ARG, "device table: reserved key");
    default:
      return set_error(HPS_ERR_ARG, "device error %d (key %llu)", e.code, k);
  }
}

// ------------------------------------------------------ small kernels ----


__global__ void iota_kernel(std::uint32_t* v, std::uint64_t n) {
  pdl_wait();
  for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       i < n; i += std::uint64_t(gridDim.x) * blockDim.x)
    v[i] = std::uint32_t(i);
}

// Per-mini-batch occurrence counts of this rank's shards and the count of
// keys it owns; range check of every key (pipeline.hpp:367-371).
__global__ void batch_count_kernel(const std::int64_t* __restrict__ off,
                                   const std::uint64_t* __restrict__ keys,
                                   std::uint64_t B, int G, int g, int J,
                                   std::uint64_t key_space,
                                   std::uint64_t* __restrict__ counts,
                                   DevError* err) {
  pdl_wait();
  __shared__ unsigned long long c[66];
  for (int i = threadIdx.x; i <= J; i += blockDim.x) c[i] = 0;
  __syncthreads();
  const std::uint64_t GJ = std::uint64_t(G) * J;
  const std::uint64_t tid = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
  const std::uint64_t nth = std::uint64_t(gridDim.x) * blockDim.x;
  for (std::uint64_t i = tid; i < B; i += nth) {
    const std::uint64_t s = i % GJ;
    if (s / J == std::uint64_t(g))
      atomicAdd(&c[s % J], (unsigned long long)(off[i + 1] - off[i]));
  }
  const std::uint64_t O = std::uint64_t(off[B]);
  if (tid == 0) counts[J + 1] = O;  // the batch's key occurrences
  unsigned long long own = 0;
  if (G == 1) {  // every key owned: the range check alone (no 64-bit division)
    for (std::uint64_t q = tid; q < O; q += nth) {
      const std::uint64_t k = keys[q];
      if (k >= key_space) raise_error(err, HPS_ERR_KEY_RANGE, k);
    }
    own = tid == 0 ? O : 0;
  } else {
    for (std::uint64_t q = tid; q < O; q += nth) {
      const std::uint64_t k = keys[q];
      if (k >= key_space) raise_error(err, HPS_ERR_KEY_RANGE, k);
      own += (k % std::uint64_t(G)) == std::uint64_t(g);
    }
  }
  atomicAdd(&c[J], own);
  __syncthreads();
  for (int i = threadIdx.x; i <= J; i += blockDim.x)
    if (c[i]) atomicAdd((unsigned long long*)&counts[i], c[i]);
}

// Shard occurrence gather: warp per shard example, occurrences numbered in
// example order (the order model.hpp sums in).
__global__ void shard_gather_kernel(ShardMap sm, const std::int64_t* __restrict__ off,
                                    const std::uint64_t* __restrict__ keys,
                                    const std::uint32_t* __restrict__ occ_off,
                                    std::uint64_t* __restrict__ kout,
                                    std::uint32_t* __restrict__ vout,
                                    std::uint32_t* __restrict__ ex_of) {
  pdl_wait();
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t w0 = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const std::uint64_t nw = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (std::uint64_t k = w0; k < sm.count; k += nw) {
    const std::uint64_t ex = sm.first + k * sm.stride;
    const std::int64_t b = off[ex], len = off[ex + 1] - b;
    const std::uint32_t o0 = occ_off[k];
    for (std::int64_t q = lane; q < len; q += 32) {
      kout[o0 + q] = keys[b + q];
      vout[o0 + q] = std::uint32_t(o0 + q);
      ex_of[o0 + q] = std::uint32_t(k);
    }
  }
}

// out[i] = rows[row_of(i)] for the parity pull (restores input order).
__global__ void scatter_rows_kernel(const std::uint32_t* __restrict__ inv,
                                    const std::uint32_t* __restrict__ pos,
                                    std::uint64_t n, int E,
                                    const float* __restrict__ rows,
                                    float* __restrict__ out) {
  pdl_wait();
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < n * E; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / E;
    const int d = int(t - i * E);
    std::uint32_t r = inv[i];
    if (pos) r = pos[r];
    out[t] = rows[std::uint64_t(r) * E + d];
  }
}

// deltas given per input key -> send order (parity push)
__global__ void permute_rows_kernel(const std::uint32_t* __restrict__ inv,
                                    const std::uint32_t* __restrict__ pos,
                                    std::uint64_t n, int E,
                                    const float* __restrict__ in,
                                    float* __restrict__ out) {
  pdl_wait();
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < n * E; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / E;
    const int d = int(t - i * E);
    std::uint32_t r = inv[i];
    if (pos) r = pos[r];
    out[std::uint64_t(r) * E + d] = in[t];
  }
}

// ---------------------------------------------------- scan functors ----

struct ShardLen {
  ShardMap sm;
  const std::int64_t* off;
  __device__ std::uint32_t operator()(std::uint64_t k) const {
    const std::uint64_t ex = sm.first + k * sm.stride;
    return std::uint32_t(off[ex + 1] - off[ex]);
  }
};
struct ShardLenEmit {
  std::uint32_t* occ_off;
  std::uint64_t n;
  __device__ void operator()(std::uint64_t k, std::uint32_t v, std::uint64_t pre) const {
    occ_off[k] = std::uint32_t(pre);
    if (k + 1 == n) occ_off[n] = std::uint32_t(pre + v);
  }
};

struct RunStart {  // first element of a run of equal keys
  const std::uint64_t* sk;
  __device__ std::uint32_t operator()(std::uint64_t p) const {
    return p == 0 || sk[p] != sk[p - 1];
  }
};
struct RunStartOwned {  // first of run and owned by rank g
  const std::uint64_t* sk;
  std::uint64_t G, g;
  __device__ std::uint32_t operator()(std::uint64_t p) const {
    return (p == 0 || sk[p] != sk[p - 1]) && (sk[p] % G == g);
  }
};
struct OwnedKey {
  const std::uint64_t* k;
  std::uint64_t G, g;
  __device__ std::uint32_t operator()(std::uint64_t q) const {
    return k[q] % G == g;
  }
};
struct CompactEmit {  // out[pre] = key (and index) for selected items
  const std::uint64_t* sk;
  const std::uint32_t* so;  // may be null
  std::uint64_t* out;
  std::uint32_t* out_idx;   // may be null
  __device__ void operator()(std::uint64_t p, std::uint32_t v, std::uint64_t pre) const {
    if (v) {
      out[pre] = sk[p];
      if (out_idx) out_idx[pre] = so ? so[p] : std::uint32_t(p);
    }
  }
};
struct LiveSlot {
  const std::uint64_t* keys;
  __device__ std::uint32_t operator()(std::uint64_t i) const { return keys[i] != kEmptyKey; }
};

struct UniqueEmit {  // inverse index + CSR segments of a sorted (key, occ) list
  const std::uint64_t* sk;
  const std::uint32_t* so;
  Count n;
  std::uint32_t* inv;
  std::uint64_t* ukeys;
  std::uint32_t* seg;
  std::uint32_t* uidv;
  const std::uint32_t* ex_of;  // occurrence -> shard example (null: none)
  std::uint32_t* exs;          // sorted position -> shard example
  __device__ void operator()(std::uint64_t p, std::uint32_t v, std::uint64_t pre) const {
    const std::uint64_t uid = pre + v - 1;
    const std::uint32_t occ = so[p];
    inv[occ] = std::uint32_t(uid);
    if (ex_of) exs[p] = ex_of[occ];
    if (v) {
      ukeys[uid] = sk[p];
      seg[uid] = std::uint32_t(p);
      uidv[uid] = std::uint32_t(uid);
    }
    const std::uint64_t nn = n.get();
    if (p + 1 == nn) seg[uid + 1] = std::uint32_t(nn);
  }
};

// --------------------------------------------------- sort / scan drivers

__global__ void context_open_kernel(std::uint32_t* context, unsigned long long* ticket) {
  pdl_wait();
  *context += 1;
  *ticket = 0;
}

// Opens a look-back context (the start of a batch body or of an API call):
// resets the device ticket counter and advances the device context counter,
// so the launches that follow bake only context-relative values.
static void open_lookback_context(Tier* t) {
  Lane& l = *t->L;
  if ((l.lb_contexts + 1) % (1u << 20) == 0)  // before the 20-bit wrap
    cudaMemsetAsync(l.status, 0, l.status_words * 8, l.st);
  ++l.lb_contexts;
  launch(t, context_open_kernel, 1, 1, 0, &l.d->context, l.ticket);
  l.tickets = 0;
  l.lb_local = 0;
}

static LookBack next_lookback(Tier* t, std::uint32_t grid) {
  Lane& l = *t->L;
  LookBack lb{l.ticket, l.tickets, ++l.lb_local, l.status, &l.d->context};
  l.tickets += grid;
  return lb;
}

template <class F, class Em>
static void tile_scan(Tier* t, F f, Em em, Count n, std::uint64_t n_upper,
                      std::uint64_t* total) {
  const std::uint32_t nb = std::max<std::uint32_t>(1, scan_tiles(n_upper));
  launch(t, scan_lookback_kernel<F, Em>, nb, kSortThreads, 0, f, em, n, next_lookback(t, nb),
         total);
}

// Digit histogram(s) + exclusive scan into t->ghist (passes > 0: 8-bit
// digits of each pass; passes == 0: owner buckets key % mod_G).
static void sort_histogram(Tier* t, const std::uint64_t* kin, Count n, std::uint64_t n_upper,
                           int passes, std::uint32_t mod_G) {
  const int np = passes ? passes : 1;
  cudaMemsetAsync(t->L->ghist, 0, std::size_t(np) * kDigits * 4, t->L->st);
  const unsigned hb = unsigned(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>((n_upper + kSortThreads - 1) / kSortThreads, kSMs * 4)));
  launch(t, onesweep_hist_kernel, hb, kSortThreads, 0, kin, n, passes, mod_G, t->L->ghist);
  launch(t, onesweep_scan_kernel, np, kDigits, 0, t->L->ghist);
}

// Stable LSD sort of n (<= n_upper) items over the low `bits` bits. Input
// (kin, vin) may alias kB/vB. Result returned through (kout, vout).
static void radix_sort(Tier* t, const std::uint64_t* kin, const std::uint32_t* vin,
                       Count n, std::uint64_t n_upper, int bits, bool values,
                       std::uint64_t** kout, std::uint32_t** vout) {
  const std::uint32_t nb = std::max<std::uint32_t>(1, sort_tiles(n_upper));
  const int passes = std::min(kMaxPasses, std::max(1, (bits + 7) / 8));
  sort_histogram(t, kin, n, n_upper, passes, 0);
  const std::uint64_t* ksrc = kin;
  const std::uint32_t* vsrc = vin;
  Lane& l = *t->L;
  std::uint64_t* kd = l.kA;
  std::uint32_t* vd = l.vA;
  for (int p = 0; p < passes; ++p) {
    const ShiftDigit dig{8 * p};
    const std::uint32_t* db = l.ghist + p * kDigits;
    if (values)
      launch(t, onesweep_pass_kernel<ShiftDigit, true>, nb, kSortThreads, 0, ksrc, vsrc, n, dig,
             db, next_lookback(t, nb), kd, vd);
    else
      launch(t, onesweep_pass_kernel<ShiftDigit, false>, nb, kSortThreads, 0, ksrc, vsrc, n, dig,
             db, next_lookback(t, nb), kd, vd);
    ksrc = kd;
    vsrc = vd;
    kd = (kd == l.kA) ? l.kB : l.kA;
    vd = (vd == l.vA) ? l.vB : l.vA;
  }
  *kout = const_cast<std::uint64_t*>(ksrc);
  *vout = const_cast<std::uint32_t*>(vsrc);
}

static int vec_of(int E) { return (E % 4 == 0) ? 4 : 1; }

// ------------------------------------------------------------ exchange --

// One exchange round (a mini-batch, or one collective API call): every
// phase of the round is tagged with the same epoch on all ranks.
// device_counter = false: the round's first kernel (owner_rank_kernel)
// increments the device counter itself.
static void begin_round(Tier* t, bool device_counter = true) {
  ++t->p2p_epoch;  // host mirror (same sequence on every rank)
  if (device_counter) launch(t, epoch_inc_kernel, 1, 1, 0, &t->dsc->epoch);
}

static void p2p_wait(Tier* t, int phase) {
  launch(t, p2p_wait_kernel, 1, 32, 0, t->ctx, t->G, t->g, phase, &t->dsc->err);
}

// Canonical sender order: node-major, device-major (hbm_ps.hpp:175-176).
static std::vector<int> canonical_senders(const Tier* t) {
  std::vector<int> v;
  for (int sn = 0; sn < t->N; ++sn)
    for (int sd = 0; sd < t->D; ++sd) v.push_back(sd * t->N + sn);
  return v;
}

// ------------------------------------------------------------- timing --

// Records the end of `phase` (the start of the next one).
static void mark(Tier* t, int phase) {
  if (!t->timing) return;
  const std::size_t i = t->ev_phase.size();
  if (i == t->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    t->evpool.push_back(e);
  }
  const int lane = int(t->L - t->lane);
  cudaStream_t s = t->L->st;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  // inside a capture the record must become an external event node
  cudaEventRecordWithFlags(t->evpool[i], s,
                           cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0);
  t->ev_phase.push_back(phase);
  t->ev_lane.push_back(lane);
}

// A phase boundary on the staging stream (lane 2).
static void mark_stage(Tier* t, int phase) {
  if (!t->timing) return;
  Lane* l = t->L;
  Lane tmp;
  tmp.st = t->st_stage;
  t->L = &tmp;
  mark(t, phase);
  t->L = l;
  t->ev_lane.back() = 2 + kGroupLanes;
}

// A phase boundary on the big-segment side stream (st3).
static void mark_big(Tier* t, int phase) {
  if (!t->timing || !t->big_side) return;
  Lane* l = t->L;
  Lane tmp;
  tmp.st = t->st3;
  t->L = &tmp;
  mark(t, phase);
  t->L = l;
  t->ev_lane.back() = 3 + kGroupLanes;
}

static void timing_begin(Tier* t) {
  t->ev_phase.clear();
  t->ev_lane.clear();
}

// After the batch is done: fold the recorded phases into acc_ms. A phase is
// the time between consecutive marks of the same lane; TOTAL spans the first
// mark to the last.
static void timing_end(Tier* t) {
  if (!t->timing || t->ev_phase.size() < 2) return;
  int last[4 + kGroupLanes];
  for (int& v : last) v = -1;
  for (std::size_t i = 0; i < t->ev_phase.size(); ++i) {
    const int ln = t->ev_lane[i], p = t->ev_phase[i];
    if (last[ln] >= 0 && p > 0 && p < HPS_TIMING_SLOTS) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t->evpool[last[ln]], t->evpool[i]);
      t->acc_ms[p] += ms;
    }
    last[ln] = int(i);
  }
  float tot = 0;
  cudaEventElapsedTime(&tot, t->evpool[0], t->evpool[t->ev_phase.size() - 1]);
  t->acc_ms[0] += tot;
}

// -------------------------------------------------------------- build --

// Build the fresh table from the working set in t->ws (count in dsc->n_ws,
// at most n_upper). staged_idx/rows: optional HostValue rows.
static int next_table(const Tier* t) { return t->cur < 0 ? 0 : (t->cur + 1) % kTables; }

static void build_table(Tier* t, std::uint64_t n_upper, const std::uint32_t* staged_idx,
                        const float* staged_rows) {
  const int nxt = next_table(t);
  const int prv = t->cur;
  launch(t, table_capacity_kernel, 1, 1, 0, (const std::uint64_t*)&t->dsc->n_ws,
         &t->dsc->cap[nxt]);
  launch(t, table_clear_kernel, grid_for(t->capmax), 256, 0, t->tkeys[nxt],
         (const std::uint64_t*)&t->dsc->cap[nxt], (const unsigned*)nullptr);
  launch(t, table_insert_kernel, grid_for(n_upper), 256, 0, (const std::uint64_t*)t->ws,
         (const std::uint64_t*)&t->dsc->n_ws, t->tkeys[nxt],
         (const std::uint64_t*)&t->dsc->cap[nxt], &t->dsc->err);
  const int V = vec_of(t->RW);
  const std::uint64_t work = n_upper * std::uint64_t(t->RW / V);
  const std::uint64_t* pcap = (prv >= 0) ? &t->dsc->cap[prv] : nullptr;
  const std::uint64_t* pk = (prv >= 0) ? t->tkeys[prv] : nullptr;
  const float* pv = (prv >= 0) ? t->tvals[prv] : nullptr;
  if (V == 4)
    launch(t, table_fill_kernel<4>, grid_for(work), 256, 0, (const std::uint64_t*)t->ws,
           (const std::uint64_t*)&t->dsc->n_ws, (const std::uint64_t*)t->tkeys[nxt],
           t->tvals[nxt], (const std::uint64_t*)&t->dsc->cap[nxt], pk, pv, pcap,
           staged_idx, staged_rows, (const float*)t->store, t->store_keys, t->RW,
           &t->dsc->carried, &t->dsc->err);
  else
    launch(t, table_fill_kernel<1>, grid_for(work), 256, 0, (const std::uint64_t*)t->ws,
           (const std::uint64_t*)&t->dsc->n_ws, (const std::uint64_t*)t->tkeys[nxt],
           t->tvals[nxt], (const std::uint64_t*)&t->dsc->cap[nxt], pk, pv, pcap,
           staged_idx, staged_rows, (const float*)t->store, t->store_keys, t->RW,
           &t->dsc->carried, &t->dsc->err);
  cudaMemcpyAsync(&t->dsc->nws_tab[nxt], &t->dsc->n_ws, 8, cudaMemcpyDeviceToDevice, t->st);
  t->prev2 = t->prev;
  t->prev = prv;
  t->cur = nxt;
  t->tab_wb[nxt] = false;  // not a train-batch table: never a store proxy
  t->tab_flushed[nxt] = false;
  t->tab_age[nxt] = ++t->builds;
  for (int k = kTables - 1; k > 0; --k) t->hist[k] = t->hist[k - 1];
  t->hist[0] = nxt;
}

// ------------------------------------------------- dedup + pull (core) --

// Dedup `n` occurrence keys (kin, occurrence ids vin; may alias kB/vB),
// partition by owner, exchange, gather rows from owners. Afterwards:
//   inv[occ] -> uid, ukeys/seg (CSR over sorted positions `so_out`),
//   pos[uid] -> send-order row (identity/null when G == 1),
//   rows[send order] filled, slots (G==1) / rslots + recv offsets (G>1).
struct PullPlan {
  std::vector<std::uint64_t> soff, roff;  // G > 1 only
  std::uint32_t* so = nullptr;            // sorted occurrence ids
  const std::uint32_t* pos = nullptr;     // null when G == 1
  std::uint64_t R = 0;                    // keys served as owner
};

static hps_status exchange_pull(Tier* t, std::uint64_t n, bool do_gather);

static hps_status dedup_pull(Tier* t, const std::uint64_t* kin, const std::uint32_t* vin,
                             Count cn, std::uint64_t n, PullPlan* plan, bool do_gather,
                             bool with_examples = false) {
  // cn: the occurrence count (host or device); n: its host upper bound
  std::uint64_t* sk = nullptr;
  std::uint32_t* so = nullptr;
  radix_sort(t, kin, vin, cn, n, t->sort_bits, true, &sk, &so);
  plan->so = so;
  tile_scan(t, RunStart{sk},
            UniqueEmit{sk, so, cn, t->inv, t->ukeys, t->seg, t->uidv,
                       with_examples ? t->ex_of : nullptr, t->exs},
            cn, n, &t->dsc->U);
  const int V = vec_of(t->E);
  if (t->G == 1) {
    mark(t, HPS_T_DEDUP);
    plan->pos = nullptr;
    if (do_gather) {
      const std::uint64_t work = n * std::uint64_t(t->E / V);
      if (V == 4)
        launch(t, table_gather_kernel<4>, grid_for(work), 256, 0,
               (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
               std::uint64_t(0), (const std::uint64_t*)t->tkeys[t->cur],
               (const float*)t->tvals[t->cur], (const std::uint64_t*)&t->dsc->cap[t->cur],
               t->rows, t->slots, t->E, t->RW, &t->dsc->err);
      else
        launch(t, table_gather_kernel<1>, grid_for(work), 256, 0,
               (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
               std::uint64_t(0), (const std::uint64_t*)t->tkeys[t->cur],
               (const float*)t->tvals[t->cur], (const std::uint64_t*)&t->dsc->cap[t->cur],
               t->rows, t->slots, t->E, t->RW, &t->dsc->err);
      mark(t, HPS_T_PULL);
    }
    return HPS_OK;
  }
  plan->pos = nullptr;
  return exchange_pull(t, n, do_gather);
}

// G > 1, the unique keys t->ukeys[0 .. dsc->U): each key's rank among the
// keys of its owner (one look-back pass that also opens the exchange round),
// then (key, uid) pairs go straight into the owners' windows over NVLink;
// rows come back in uid order into t->rows.
static hps_status exchange_pull(Tier* t, std::uint64_t n, bool do_gather) {
  const int V = vec_of(t->E);
  {
    const std::uint32_t nb = std::max<std::uint32_t>(
        1, std::uint32_t((n + kRankTile - 1) / kRankTile));
    launch(t, owner_rank_kernel, nb, kRankThreads, 0, (const std::uint64_t*)t->ukeys,
           (const std::uint64_t*)&t->dsc->U, t->G, next_lookback(t, nb), t->orank, t->otot,
           &t->dsc->epoch, &t->dsc->n_long);
  }
  launch(t, p2p_send_keys_kernel, grid_for(n, 256, kSMs * 4), 256, 0, t->ctx, t->G, t->g, t->slot,
         (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
         (const std::uint32_t*)t->orank, (const std::uint64_t*)t->otot, t->done_ctr);
  // the keys wait is folded into serve_rows (each CTA polls the flags) unless
  // there is no gather or HPS_FOLD_WAIT=0
  const bool fold = do_gather && t->fold_wait;
  if (!fold) p2p_wait(t, kPhKeys);
  mark(t, HPS_T_DEDUP);
  if (do_gather) {
    const std::uint64_t work = t->Omax * std::uint64_t(t->E / V);
    auto k = V == 4 ? p2p_serve_rows_kernel<4> : p2p_serve_rows_kernel<1>;
    launch(t, k, grid_for(work, 256, kSMs * 4), 256, 0, t->ctx, t->G, t->g, t->slot,
           (const std::uint64_t*)t->tkeys[t->cur], (const float*)t->tvals[t->cur],
           (const std::uint64_t*)&t->dsc->cap[t->cur], t->w_rslots, t->E, t->RW, t->done_ctr,
           &t->dsc->served, &t->dsc->err, fold ? int(kPhKeys) : -1, int(kPhRows));
    p2p_wait(t, kPhRows);
    mark(t, HPS_T_PULL);
  }
  return HPS_OK;
}

// Owner apply of the pushed deltas in canonical sender order (G > 1): the
// delta rows go straight into the owners' windows; each owner applies the
// sources' segments in (node, device) order with the slots cached at pull.
static hps_status push_apply(Tier* t) {
  const int V = vec_of(t->E);
  const std::uint64_t work = t->Omax * std::uint64_t(t->E / V);
  if (V == 4)
    launch(t, p2p_send_deltas_kernel<4>, grid_for(work, 256, kSMs * 4), 256, 0, t->ctx, t->G,
           t->g, t->slot, (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
           (const std::uint32_t*)t->orank, (const float*)t->deltas, t->E, t->done_ctr);
  else
    launch(t, p2p_send_deltas_kernel<1>, grid_for(work, 256, kSMs * 4), 256, 0, t->ctx, t->G,
           t->g, t->slot, (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
           (const std::uint32_t*)t->orank, (const float*)t->deltas, t->E, t->done_ctr);
  if (!t->fold_wait) p2p_wait(t, kPhDeltas);
  bool first = t->fold_wait;  // the first apply waits for every source's deltas
  auto k = V == 4 ? p2p_apply_kernel<4> : p2p_apply_kernel<1>;
  for (int src : canonical_senders(t)) {
    launch(t, k, grid_for(t->slot * std::uint64_t(t->E / V), 256, kSMs * 2), 256, 0, t->ctx, t->g,
           src, t->slot, (const std::uint32_t*)t->w_rslots, t->tvals[t->cur], t->opt, t->G,
           first ? int(kPhDeltas) : -1, &t->dsc->err, 0);
    first = false;
  }
  return HPS_OK;
}

// Dense sync of t->dgrad (replica buffers) + update of t->dense.
static hps_status dense_sync_update(Tier* t, bool apply) {
  const std::uint64_t nw = std::uint64_t(t->md.nw);
  if (t->G == 1) {
    launch(t, dense_update_kernel, grid_for(nw), 256, 0, t->dense,
           (const float*)t->dgrad, nw, t->N, t->D, t->cfg.learning_rate, int(apply),
           (float*)nullptr, &t->dsc->err, (const float*)nullptr,
           (const unsigned long long*)nullptr);
    return HPS_OK;
  }
  // replicas all-gathered over NVLink, then the canonical f64 sum (det and
  // fast modes alike: the canonical order costs nothing extra here)
  launch(t, p2p_send_dense_kernel, grid_for(nw * t->G), 256, 0, t->ctx, t->G, t->g, nw,
         (const float*)t->dgrad, t->done_ctr);
  launch(t, p2p_dense_update_kernel, 1, 256, 0, t->ctx, t->G, t->g, t->N, t->D, nw, t->dense,
         t->cfg.learning_rate, int(apply), (float*)nullptr, &t->dsc->err, int(kPhDense));
  return HPS_OK;
}

// One tcgen05 GEMM (mlp.cuh) on stream s; BN by N, split-K over grid.z.
static void launch_gemm(Tier* t, cudaStream_t s, GemmArgs g, int splits = 1) {
  splits = std::max(1, splits);
  const int kps = ((g.K + splits - 1) / splits + kGemmBK - 1) / kGemmBK * kGemmBK;
  splits = (g.K + kps - 1) / kps;
  g.k_per_split = kps;
  g.split3 = t->gemm_split3 ? 1 : 0;
  auto smem = [&](int bn) { return gemm_smem(bn, g.split3 != 0); };
  const unsigned gm = unsigned((g.M + kGemmBM - 1) / kGemmBM);
  // N > 64 in 128-wide tiles (256 would halve the CTAs and, with the 3xTF32
  // split, fit only two pipeline stages: measured 78 us vs ~30 us per c4 GEMM)
  if (g.N > 64) {
    launch_on(t, s, umma_gemm_kernel<128>, dim3(gm, unsigned((g.N + 127) / 128), unsigned(splits)),
              kGemmThreads, smem(128), g);
  } else if (g.N > 32) {
    launch_on(t, s, umma_gemm_kernel<64>, dim3(gm, 1, unsigned(splits)), kGemmThreads, smem(64), g);
  } else {
    launch_on(t, s, umma_gemm_kernel<32>, dim3(gm, 1, unsigned(splits)), kGemmThreads, smem(32), g);
  }
}

// Forward + backward of one mini-batch shard on the wide path (mlp.cuh): the
// activations and the dL/dx records on the body stream, the weight gradients
// on st2 beside the sparse reduce (fork recorded after dX, joined by the
// caller through t->join), all into t->dgrad in the reference layout.
static hps_status enqueue_wide(Tier* t, const ShardMap& sm, std::uint64_t n,
                               const std::int64_t* goff, const std::uint32_t* occ_row,
                               const float* rows, int rstride, const std::uint8_t* dlab) {
  const ModelDims& md = t->md;
  const int L = md.L, E = t->E;
  launch(t, wide_embed_kernel, grid_for(n * 32), 256, 0, sm, goff,
         (const std::uint32_t*)t->occ_off, occ_row, rows, rstride, E, t->wX);
  const float* hin = t->wX;
  for (int l = 0; l + 1 < L; ++l) {  // hidden layers: Z = H W^T + b, relu
    const int out = md.dims[l], in = md.ins[l];
    const float* W = t->dense + md.offs[l];
    GemmArgs g{};
    g.M = int(n), g.N = out, g.K = in;
    g.A = hin, g.a_m = in, g.a_k = 1;
    g.B = W, g.b_n = in, g.b_k = 1;
    g.epi = kEpiBiasRelu, g.D = t->wH[l], g.ldd = out, g.bias = W + std::int64_t(in) * out;
    launch_gemm(t, t->st, g);
    hin = t->wH[l];
  }
  {  // output layer, sigmoid, loss, output delta -> the last hidden layer's dZ
    const int K = md.ins[L - 1];
    const float* W = t->dense + md.offs[L - 1];
    launch(t, wide_head_kernel, grid_for(n * 32), 256, 0, sm, K, W, W + K, hin, dlab, t->wdz,
           t->wdZ[L - 2], &t->dsc->loss, &t->dsc->err);
  }
  for (int l = L - 2; l >= 0; --l) {  // dZ_{l-1} = (dZ_l W_l) .* [H_{l-1} > 0]; dX at l = 0
    const int out = md.dims[l], in = md.ins[l];
    GemmArgs g{};
    g.M = int(n), g.N = in, g.K = out;
    g.A = t->wdZ[l], g.a_m = out, g.a_k = 1;
    g.B = t->dense + md.offs[l], g.b_n = 1, g.b_k = in;
    if (l > 0) {
      g.epi = kEpiMask, g.D = t->wdZ[l - 1], g.ldd = in, g.mask = t->wH[l - 1], g.ldm = in;
    } else {
      g.epi = kEpiF64, g.Dd = t->DX, g.ldd = in;
    }
    launch_gemm(t, t->st, g);
  }
  mark(t, HPS_T_FWDBWD);
  // weight gradients beside the sparse reduce
  HPS_CUDA(cudaEventRecord(t->fork, t->st));
  HPS_CUDA(cudaStreamWaitEvent(t->st2, t->fork, 0));
  {
    const int K = md.ins[L - 1];
    launch_on(t, t->st2, wide_head_grad_kernel, unsigned(K + 1), 256, 0, n, K,
              (const float*)t->wdz, (const float*)t->wH[L - 2], t->dgrad + md.offs[L - 1]);
  }
  for (int l = L - 2; l >= 0; --l) {  // [dW_l | db_l] = dZ_l^T [H_{l-1} | 1] / n
    const int out = md.dims[l], in = md.ins[l];
    GemmArgs g{};
    g.M = out, g.N = in + 1, g.K = int(n);
    g.A = t->wdZ[l], g.a_m = 1, g.a_k = out;
    g.B = l > 0 ? t->wH[l - 1] : t->wX, g.b_n = 1, g.b_k = in, g.b_ones_col = 1;
    g.epi = kEpiStore, g.D = t->wP, g.ldd = in + 1;
    const int bn = g.N > 64 ? 128 : (g.N > 32 ? 64 : 32);
    const int tiles = ((out + kGemmBM - 1) / kGemmBM) * ((g.N + bn - 1) / bn);
    int splits = std::max(1, kSMs / tiles);
    splits = int(std::min<std::uint64_t>(std::uint64_t(splits), (n + kGemmBK - 1) / kGemmBK));
    while (splits > 1 && std::uint64_t(splits) * out * (in + 1) > t->wP_cap) --splits;
    const int kps = ((int(n) + splits - 1) / splits + kGemmBK - 1) / kGemmBK * kGemmBK;
    splits = (int(n) + kps - 1) / kps;
    launch_gemm(t, t->st2, g, splits);
    float* gW = t->dgrad + md.offs[l];
    launch_on(t, t->st2, wide_wgrad_reduce_kernel, grid_for(std::uint64_t(out) * (in + 1)), 256, 0,
              (const float*)t->wP, splits, out, in, n, gW, gW + std::int64_t(in) * out);
  }
  HPS_CUDA(cudaEventRecord(t->join, t->st2));
  return HPS_OK;
}

// Segment-length routing of the sparse reduce: <= kLongSeg in-order by one
// thread per (key, 4 dims), longer ones split into fuse_chunk(E)-occurrence
// chunks over CTAs (big_fused_kernel).
//
// The big-segment path's preparation, on st3 beside fwd/bwd: list the keys
// with segments over kLongSeg (big_classify_kernel), plan their (key, chunk)
// items, reset the fused kernel's flags and ticket.
// zero_kernel over (pointer, bytes) regions (bytes a multiple of 4) on s.
static void zero_on(Tier* t, cudaStream_t s,
                    std::initializer_list<std::pair<void*, std::size_t>> regions) {
  ZeroList z{};
  int r = 0;
  for (const auto& pr : regions) {
    z.p[r] = reinterpret_cast<std::uint32_t*>(pr.first);
    z.n[r] = std::uint32_t(pr.second / 4);
    ++r;
  }
  for (; r < kZeroRegions; ++r) {
    z.p[r] = nullptr;
    z.n[r] = 0;
  }
  launch_on(t, s, zero_kernel, 1, 128, 0, z);
}

static hps_status launch_big_plan(Tier* t, std::uint64_t u_upper, const std::uint64_t* U,
                                  const std::uint32_t* seg) {
  unsigned long long* nb = &t->dsc->n_big;
  cudaStream_t bs = t->big_side ? t->st3 : t->st;
  // the counters and the fused kernel's ticket (its previous use, the last
  // mini-batch's big_fused_kernel, ran earlier on this stream)
  zero_on(t, bs, {{nb, 8}, {&t->dsc->n_mid, 8}, {t->fuse_ticket, 8}});
  launch_on(t, bs, big_classify_kernel, grid_for(std::max<std::uint64_t>(u_upper, 1)), 256, 0,
            U, seg, t->big_list, nb, t->short_max, t->mid_max, t->mid_list, &t->dsc->n_mid);
  launch_on(t, bs, big_plan_kernel, 1, 1024, 0, fuse_chunk(t->E),
            (const std::uint32_t*)t->big_list, (const unsigned long long*)nb, seg, t->chunk_off,
            &t->dsc->n_items, t->item_key, t->item_chunk, &t->dsc->big_keys, &t->dsc->max_chunks,
            &t->dsc->big_occ);
  return HPS_OK;
}

// The sparse segment-reduce: short segments on the body stream, big ones
// (planned by launch_big_plan) in one fused pass over CTAs on st3 (ticket
// order). The caller forks st3 after fwd/bwd and joins it (join3).
static hps_status launch_sparse_delta(Tier* t, std::uint64_t n, const std::uint32_t* pos,
                                      std::uint64_t u_upper, const std::uint64_t* U,
                                      const std::uint32_t* seg, const std::uint32_t* exs,
                                      const std::uint32_t* apply_slot = nullptr,
                                      bool short_side = false) {
  // apply_slot non-null (one rank, the keys' table slots known): the deltas
  // go straight into the current table, no delta rows and no apply launch
  const DeltaOut dout{t->deltas, pos, apply_slot, apply_slot ? t->tvals[t->cur] : nullptr,
                      t->opt};
  const int E = t->E;
  if (E > 256) return set_error(HPS_ERR_ARG, "embedding_dim <= 256");
  const float lr = t->cfg.learning_rate;
  const double* DX = t->DX;
  cudaStream_t bs = t->big_side ? t->st3 : t->st;
  // medium segments: exact warp chains on st4, beside the big and short paths
  // (after the classification on bs and fwd/bwd's dL/dx)
  cudaStream_t ms = t->big_side ? t->st4 : t->st;
  if (t->big_side) {
    HPS_CUDA(cudaEventRecord(t->fork4, bs));
    HPS_CUDA(cudaStreamWaitEvent(ms, t->fork4, 0));
  }
  const bool mid_cert = t->mid_cert && (E == 4 || E == 8 || E == 16 || E == 32);
  if (t->mid_max > t->short_max && mid_cert) {
    auto mk = E == 4 ? sparse_mid_cert_kernel<4>
                     : (E == 8 ? sparse_mid_cert_kernel<8>
                               : (E == 16 ? sparse_mid_cert_kernel<16> : sparse_mid_cert_kernel<32>));
    launch_on(t, ms, mk, kSMs * 2, 32 * kMidCertWarps, mid_cert_smem(), n,
              (const unsigned long long*)&t->dsc->n_mid, (const std::uint32_t*)t->mid_list, seg,
              exs, dout, DX, &t->dsc->mid_keys, &t->dsc->fallbacks, int(t->wide));
  } else if (t->mid_max > t->short_max) {
    const int rpi = E <= 8 ? 4 : (E <= 16 ? 2 : 1);
    auto mk = rpi == 4 ? sparse_mid_kernel<4> : (rpi == 2 ? sparse_mid_kernel<2> : sparse_mid_kernel<1>);
    launch_on(t, ms, mk, kSMs * 4, 32 * kMidWarps, mid_smem(rpi), E, n,
              (const unsigned long long*)&t->dsc->n_mid, (const std::uint32_t*)t->mid_list, seg,
              exs, dout, DX, &t->dsc->mid_keys);
  }
  if (t->big_side) HPS_CUDA(cudaEventRecord(t->join4, ms));
  mark_big(t, -1);
  launch_on(t, bs, big_fused_kernel, kSMs * 4, kFuseThreads, 0, E, lr, n,
            (const std::uint32_t*)t->big_list, (const unsigned long long*)&t->dsc->n_big,
            (const std::uint32_t*)t->chunk_off, (const unsigned long long*)&t->dsc->n_items,
            (const std::uint32_t*)t->item_key, (const std::uint32_t*)t->item_chunk, seg, exs,
            dout, DX, t->chunk_tot, t->fuse_ticket, t->key_done, &t->dsc->fallbacks);
  mark_big(t, HPS_T_BIGFUSED);
  HPS_CUDA(cudaEventRecord(t->join3, bs));
  // DPT dims per thread: 4 when E allows 32-byte row loads (8 measured 1-2%
  // slower in the pipelined c2 step: fewer threads in flight; HPS_SHORT_DPT=8)
  const int dpt = t->short_dpt ? t->short_dpt : ((E % 4 == 0) ? 4 : 1);
  auto sk = dpt == 8 ? sparse_short_kernel<8>
                     : (dpt == 4 ? sparse_short_kernel<4> : sparse_short_kernel<1>);
  // grid-stride over the keys, capped (HPS_SHORT_GRID) so the medium / hot-key
  // reduces and the dense gradient, forked at the same point, find SM slots
  // at once instead of after this kernel's last wave
  const unsigned sg = grid_for(std::max<std::uint64_t>(u_upper, 1) * (E / dpt), 256,
                               t->short_grid ? t->short_grid : kSMs * 32);
  if (short_side) {  // (the caller keeps st for the dense gradient and joins all)
    launch_on(t, t->st2, sk, sg, 256, 0, E, t->short_max, n, U, seg, exs, dout, DX,
              &t->dsc->pulled);
    HPS_CUDA(cudaEventRecord(t->join, t->st2));
    return HPS_OK;
  }
  launch(t, sk, sg, 256, 0, E, t->short_max, n, U, seg, exs, dout, DX, &t->dsc->pulled);
  HPS_CUDA(cudaStreamWaitEvent(t->st, t->join3, 0));
  if (t->big_side) HPS_CUDA(cudaStreamWaitEvent(t->st, t->join4, 0));
  return HPS_OK;
}

// Exported window of this rank + the peers' windows (p2p.cuh). Ranks in
// other processes are mapped through CUDA IPC handles; ranks in this process
// through peer access. The window descriptors are all-gathered with NCCL.
static hps_status setup_p2p(Tier* t, std::uint64_t S) {
  const int G = t->G;
  if (G > kMaxRanks) return set_error(HPS_ERR_ARG, "at most %d GPUs per tier", kMaxRanks);
  const std::uint64_t E = std::uint64_t(t->E), nw = std::uint64_t(t->md.nw);
  t->slot = t->Omax;
  auto al = [](std::uint64_t b) { return (b + 255) & ~std::uint64_t(255); };
  const std::uint64_t o_flags = 0;
  const std::uint64_t o_rows = o_flags + al(G * kPhases * 8);
  const std::uint64_t o_par = o_rows + al(S * E * 4);  // two parity copies follow
  const std::uint64_t p_keys = 0;
  const std::uint64_t p_uids = p_keys + al(G * t->slot * 8);
  const std::uint64_t p_hdr = p_uids + al(G * t->slot * 4);
  const std::uint64_t p_deltas = p_hdr + al(G * 2 * 8);
  const std::uint64_t p_dense = p_deltas + al(G * t->slot * E * 4);
  const std::uint64_t par_bytes = p_dense + al(G * nw * 4);
  const std::uint64_t total = o_par + 2 * par_bytes;
  HPS_CUDA(cudaMalloc(&t->win_base, total));
  t->allocs.push_back(t->win_base);
  HPS_CUDA(cudaMemset(t->win_base, 0, total));
  char* b = static_cast<char*>(t->win_base);
  t->w_flags = reinterpret_cast<std::uint64_t*>(b + o_flags);
  t->rows = reinterpret_cast<float*>(b + o_rows);
  for (int par = 0; par < 2; ++par) {
    char* pb = b + o_par + par * par_bytes;
    t->w_keys_p[par] = reinterpret_cast<std::uint64_t*>(pb + p_keys);
    t->w_hdr_p[par] = reinterpret_cast<std::uint64_t*>(pb + p_hdr);
    t->w_deltas_p[par] = reinterpret_cast<float*>(pb + p_deltas);
    t->w_dense_p[par] = reinterpret_cast<float*>(pb + p_dense);
  }
  HPS_TRY(dalloc(t, &t->w_rslots, G * t->slot));
  HPS_TRY(dalloc(t, &t->done_ctr, 1));
  HPS_CUDA(cudaMemset(t->done_ctr, 0, 4));
  struct Info {
    cudaIpcMemHandle_t h;
    std::uint64_t base;
    std::int32_t pid, dev;
  };
  Info mine{};
  HPS_CUDA(cudaIpcGetMemHandle(&mine.h, t->win_base));
  mine.base = reinterpret_cast<std::uint64_t>(t->win_base);
  mine.pid = std::int32_t(getpid());
  mine.dev = t->cfg.cuda_device;
  std::vector<Info> all(G);
  char* dinfo = nullptr;
  HPS_CUDA(cudaMalloc(&dinfo, sizeof(Info) * (G + 1)));
  HPS_CUDA(cudaMemcpy(dinfo, &mine, sizeof(Info), cudaMemcpyHostToDevice));
  ncclResult_t r = nccl().AllGather(dinfo, dinfo + sizeof(Info), sizeof(Info), ncclUint8, t->comm,
                                    t->st);
  if (r != ncclSuccess) {
    cudaFree(dinfo);
    return set_error(HPS_ERR_NCCL, "nccl: window exchange: %s", nccl().GetErrorString(r));
  }
  HPS_CUDA(cudaStreamSynchronize(t->st));
  HPS_CUDA(cudaMemcpy(all.data(), dinfo + sizeof(Info), sizeof(Info) * G, cudaMemcpyDeviceToHost));
  cudaFree(dinfo);
  for (int p = 0; p < G; ++p) {
    char* base = nullptr;
    if (p == t->g) {
      base = b;
    } else if (all[p].pid == mine.pid) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(all[p].dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return set_error(HPS_ERR_CUDA, "cuda: peer access %d->%d: %s", mine.dev, all[p].dev,
                         cudaGetErrorString(e));
      cudaGetLastError();
      base = reinterpret_cast<char*>(all[p].base);
    } else {
      void* q = nullptr;
      HPS_CUDA(cudaIpcOpenMemHandle(&q, all[p].h, cudaIpcMemLazyEnablePeerAccess));
      t->ipc_opened.push_back(q);
      base = static_cast<char*>(q);
    }
    for (int par = 0; par < 2; ++par) {
      char* pb = base + o_par + par * par_bytes;
      PeerWindows& w = t->ctx.par[par];
      w.keys[p] = reinterpret_cast<std::uint64_t*>(pb + p_keys);
      w.uids[p] = reinterpret_cast<std::uint32_t*>(pb + p_uids);
      w.hdr[p] = reinterpret_cast<std::uint64_t*>(pb + p_hdr);
      w.deltas[p] = reinterpret_cast<float*>(pb + p_deltas);
      w.dense[p] = reinterpret_cast<float*>(pb + p_dense);
      w.flags[p] = reinterpret_cast<std::uint64_t*>(base + o_flags);
      w.rows[p] = reinterpret_cast<float*>(base + o_rows);
    }
  }
  {
    const char* v = std::getenv("HPS_CTA_FENCE");
    const int sys = v && std::strcmp(v, "sys") == 0;
    t->ctx.par[0].cta_sys_fence = t->ctx.par[1].cta_sys_fence = sys;
  }
  t->ctx.epoch = &t->dsc->epoch;
  begin_round(t);  // round 1 (flags start at 0)
  return HPS_OK;
}

// ------------------------------------------------- the per-batch body --

inline std::uint64_t shape_bound(std::uint64_t x) {
  std::uint64_t p = 4096;
  while (p < x) p <<= 1;
  return p;
}

static unsigned prep_grid_of(const Tier* t, unsigned g) {
  return t->prep_grid ? std::min(g, t->prep_grid) : g;
}

// Start of mini-batch j's region in the per-table grouping pools: the sum of
// the earlier mini-batches' shape bounds (stable per shape, so captured
// graphs hold across batches).
static std::uint64_t group_region(const BatchShape& sh, int j) {
  std::uint64_t r = 0;
  for (int i = 0; i < j; ++i) r += sh.mb_bound[i];
  return r;
}

// Mini-batch dedup of every shard of the batch by slot grouping (group.cuh),
// on the prep lane: it depends only on the keys, so batch b+1's grouping runs
// beside batch b's body. Outputs go to the table's pools (g_*[tb]).
static hps_status enqueue_grouping(Tier* T, const BatchShape& sh, const BatchPlan& bp,
                                   GroupState& g, int j0, int j1, DevError* err,
                                   const cudaEvent_t* mb_done = nullptr) {
  const int G = T->G, J = T->J, tb = bp.tb;
  const std::uint64_t B = sh.B, GJ = std::uint64_t(G) * J;
  const std::int64_t* doff = T->b_off[bp.sp];
  const std::uint64_t* dkeys = T->b_keys[bp.sp];
  Lane& l = *T->L;
  const std::uint32_t pcap = std::uint32_t(T->part_cap);
  for (int j = j0; j < j1 && j < J; ++j) {
    const std::uint64_t s = std::uint64_t(T->g) * J + j;
    const std::uint64_t n = s < B ? (B - s - 1) / GJ + 1 : 0;
    const ShardMap sm{s, GJ, n};
    const std::uint64_t ob = sh.mb_bound[j], r0 = group_region(sh, j);
    std::uint32_t* seg = T->g_segb[tb] + r0 + j;  // U+1 entries per region
    std::uint32_t* exs = T->g_exsb[tb] + r0;
    std::uint32_t* uids = T->g_uidb[tb] + r0;
    std::uint32_t* segocc = T->g_segocc[tb] + r0;  // (positions are per mini-batch)
    unsigned long long* U = &T->dsc->Ug[tb][j];
    zero_on(T, l.st, {{U, 8}, {g.gn, 4 * sizeof(unsigned long long)}});
    if (!n) {
      if (mb_done) HPS_CUDA(cudaEventRecord(mb_done[j], l.st));
      continue;
    }
    const std::uint64_t warps = ((n + 31) / 32) * kGroupPosGroups;
    // slot space: the batch table (G == 1: it holds every key) or the
    // rank's request table (G > 1)
    const std::uint64_t* gk = G == 1 ? T->tkeys[tb] : T->rq_keys[tb];
    const std::uint64_t* gc = G == 1 ? &T->dsc->cap[tb] : &T->dsc->rq_capv;
    launch(T, group_probe_kernel, prep_grid_of(T, grid_for(warps * 32)), 256, 0, sm, doff, dkeys, gk, gc, g.gcnt,
           g.slot_uid, g.part_slot, pcap, g.part_n, T->g_occslot[tb], T->g_tick[tb], T->g_exof[tb],
           err, G == 1);
    launch(T, group_compact_kernel, prep_grid_of(T, grid_for(ob)), 256, 0, (const std::uint32_t*)g.part_n,
           (const std::uint32_t*)g.part_slot, pcap, g.part_base, uids, U);
    const Count Uc{reinterpret_cast<const std::uint64_t*>(U), 0};
    tile_scan(T, UidCount{uids, g.gcnt}, SegEmit{seg, Uc}, Uc, ob, &l.d->total);
    const std::uint32_t words = std::uint32_t((n + 31) / 32);
    const std::size_t wsmem = std::size_t(kGroupWarpThreads / 32) * 2 * words * 4;
    if (T->group_fused) {
      // place also resets the slot counters and lists the longer segments;
      // one launch then orders every segment
      launch(T, group_place_kernel, prep_grid_of(T, grid_for(n * 32)), 256, 0, sm, doff,
             (const std::uint32_t*)T->g_occslot[tb], (const std::uint32_t*)T->g_tick[tb],
             (const std::uint32_t*)g.slot_uid, pcap, (const std::uint32_t*)g.part_base,
             (const std::uint32_t*)seg, segocc, G == 1 ? nullptr : T->g_inv[tb], g.gcnt, g.part_n,
             g.g_long, &g.gn[0], g.g_huge, &g.gn[2]);
      launch(T, group_sort_kernel, kSMs * 2, kGroupSortThreads,
             std::size_t(kGroupSortThreads / 32) * 2 * words * 4,
             (const unsigned long long*)U, (const std::uint32_t*)seg, (const std::uint32_t*)segocc,
             (const std::uint32_t*)T->g_exof[tb], words, exs,
             (const unsigned long long*)&g.gn[0], (const std::uint32_t*)g.g_long,
             (const unsigned long long*)&g.gn[2], (const std::uint32_t*)g.g_huge);
    } else {
    launch(T, group_place_kernel, prep_grid_of(T, grid_for(n * 32)), 256, 0, sm, doff,
           (const std::uint32_t*)T->g_occslot[tb], (const std::uint32_t*)T->g_tick[tb],
           (const std::uint32_t*)g.slot_uid, pcap, (const std::uint32_t*)g.part_base,
           (const std::uint32_t*)seg, segocc, G == 1 ? nullptr : T->g_inv[tb],
           (std::uint32_t*)nullptr, (std::uint32_t*)nullptr, (std::uint32_t*)nullptr,
           (unsigned long long*)nullptr, (std::uint32_t*)nullptr, (unsigned long long*)nullptr);
    launch(T, group_order_kernel, prep_grid_of(T, grid_for(ob)), 256, 0, (const unsigned long long*)U,
           (const std::uint32_t*)seg, segocc, (const std::uint32_t*)T->g_exof[tb],
           (const std::uint32_t*)uids, g.gcnt, exs, g.g_long, &g.gn[0], g.g_huge,
           &g.gn[2], g.part_n);
    launch(T, group_warp_kernel, kSMs * 4, kGroupWarpThreads, wsmem,
           (const unsigned long long*)&g.gn[0], (const std::uint32_t*)g.g_long,
           (const std::uint32_t*)seg, (const std::uint32_t*)segocc,
           (const std::uint32_t*)T->g_exof[tb], words, exs, g.g_dup, &g.gn[1]);
    launch(T, group_cta_kernel, kSMs, kGroupThreads, std::size_t(2) * words * 4,
           (const unsigned long long*)&g.gn[2], (const std::uint32_t*)g.g_huge,
           (const std::uint32_t*)seg, (const std::uint32_t*)segocc,
           (const std::uint32_t*)T->g_exof[tb], words, exs, g.g_dup, &g.gn[1]);
    launch(T, group_dup_kernel, kSMs, kGroupThreads, 0,
           (const unsigned long long*)&g.gn[1], (const std::uint32_t*)g.g_dup,
           (const std::uint32_t*)seg, (const std::uint32_t*)segocc,
           (const std::uint32_t*)T->g_exof[tb], exs);
    }
    if (G > 1 && T->xfuse && T->xprep) {
      // the fused exchange's keys of this mini-batch, off the body's path:
      // unique keys in uid order and their owner ranks (no round opened here)
      std::uint64_t* xk = T->pxukeys[tb] + r0;
      launch(T, uid_keys_kernel, grid_for(ob), 256, 0, (const std::uint32_t*)uids,
             (const std::uint64_t*)T->rq_keys[tb], (const unsigned long long*)U, xk,
             &T->dsc->xscratch[0]);
      const std::uint32_t nb =
          std::max<std::uint32_t>(1, std::uint32_t((ob + kRankTile - 1) / kRankTile));
      launch(T, owner_rank_kernel, nb, kRankThreads, 0, (const std::uint64_t*)xk,
             (const std::uint64_t*)U, T->G, next_lookback(T, nb), T->pxorank[tb] + r0,
             T->pxotot[tb] + std::uint64_t(j) * kMaxRanks, &T->dsc->xscratch[1],
             &T->dsc->xscratch[2]);
    }
    if (mb_done) HPS_CUDA(cudaEventRecord(mb_done[j], l.st));
  }
  return HPS_OK;
}

// Whether the prep sorts the working set by key (Tier::ws_sort).
static bool ws_sorted(const Tier* T) { return T->ws_sort < 0 ? T->store_on_host : T->ws_sort != 0; }

// Prep of one batch (lane 1, beside the previous batch's body): the sort-free
// build of its table. Exact distinct count through a scratch set (it fixes
// the capacity, hence the layout), ordered probing of the raw owned
// occurrences (duplicates stop on their own key; ordered probing is
// history-independent, so the layout equals ascending insertion,
// hbm_ps.hpp:69-98), the distinct keys with their slots in ascending key
// order (compact + sort), then every row that is not a carry-over: from the
// table two builds back when it holds the key, else the value store.
// Enqueue-only (capturable).
static hps_status enqueue_prep(Tier* T, const BatchShape& sh, const BatchPlan& bp) {
  const int G = T->G, E = T->E, tb = bp.tb;
  Lane& l = *T->L;
  const std::uint64_t* dkeys = T->b_keys[bp.sp];
  std::uint64_t* nws = &T->dsc->nws_tab[tb];
  std::uint64_t* cap = &T->dsc->cap[tb];
  DevError* perr = &T->dsc->perr[tb];
  mark(T, -1);
  zero_on(T, l.st, {{perr, sizeof(DevError)}, {nws, 8}, {&T->dsc->carried_tab[tb], 8},
                    {&T->dsc->stored_tab[tb], 8}, {&T->dsc->spec_fail, 4}});
  const unsigned gk = prep_grid_of(T, grid_for(sh.batch_bound, 256, kSMs * 8));
  const std::uint64_t cap_bound = table_capacity(sh.own_bound);
  // speculative build at the previous table's capacity (a steady workload
  // keeps it), counting the distinct keys; the check redoes the build at the
  // counted capacity when it differs — the layout is the same either way
  launch(T, table_guess_kernel, 1, 1, 0, bp.tp >= 0 ? (const std::uint64_t*)&T->dsc->cap[bp.tp]
                                                    : (const std::uint64_t*)nullptr,
         std::min(cap_bound, T->capmax), cap);  // (the shape bound may exceed the buffers)
  launch(T, table_clear_kernel, grid_for(cap_bound), 256, 0, T->tkeys[tb],
         (const std::uint64_t*)cap, (const unsigned*)nullptr);
  launch(T, table_insert_dedup_kernel, gk, 256, 0, (const std::int64_t*)T->b_off[bp.sp], sh.B,
         dkeys, std::uint64_t(G), std::uint64_t(T->g), T->tkeys[tb], (const std::uint64_t*)cap,
         perr, (unsigned long long*)nws, &T->dsc->spec_fail, (const unsigned*)nullptr);
  // (a speculative table that fills up stops counting, so its
  // count cannot size the redo; that redo runs at the bound's capacity and a
  // second check re-sizes it from the then exact count)
  const std::uint64_t fallback = std::min(cap_bound, T->capmax);
  for (int pass = 0; pass < 2; ++pass) {
    launch(T, table_spec_check_kernel, 1, 1, 0, (unsigned long long*)nws, cap,
           &T->dsc->spec_fail, &T->dsc->redo, fallback);
    launch(T, table_clear_kernel, grid_for(cap_bound), 256, 0, T->tkeys[tb],
           (const std::uint64_t*)cap, (const unsigned*)&T->dsc->redo);
    launch(T, table_insert_dedup_kernel, gk, 256, 0, (const std::int64_t*)T->b_off[bp.sp], sh.B,
           dkeys, std::uint64_t(G), std::uint64_t(T->g), T->tkeys[tb], (const std::uint64_t*)cap,
           perr, (unsigned long long*)nws,
           pass == 0 ? &T->dsc->spec_fail : (unsigned*)nullptr, (const unsigned*)&T->dsc->redo);
  }
  // the table's keys are final: the mini-batches' grouping forks onto lane 2
  // and runs beside the rest of the build (joined at the end of the prep)
  if (bp.grouped) {
    if (G > 1) {  // the request table: every key of this rank's shards
      HPS_CUDA(cudaMemsetAsync(T->rq_keys[tb], 0xFF, T->rq_cap * 8, l.st));
      launch(T, rq_insert_kernel, grid_for(sh.B * 32), 256, 0, T->b_off[bp.sp],
             (const std::uint64_t*)dkeys, sh.B, G, T->g, T->J, T->rq_keys[tb],
             (const std::uint64_t*)&T->dsc->rq_capv);
    }
    HPS_CUDA(cudaEventRecord(T->g_fork, l.st));
    const int np = T->prep_group_lanes;  // lanes 2 .. 2 + np - 1, mini-batches alternating
    for (int i = 0; i < np; ++i) HPS_CUDA(cudaStreamWaitEvent(T->lane[2 + i].st, T->g_fork, 0));
    hps_status st = HPS_OK;
    for (int j = 0; j < bp.prep_mbs && st == HPS_OK; ++j) {
      T->L = &T->lane[2 + j % np];
      st = enqueue_grouping(T, sh, bp, T->gs[j % np], j, j + 1, perr);
    }
    T->L = &T->lane[2];
    if (st == HPS_OK) mark(T, HPS_T_DEDUP);
    T->L = &l;
    HPS_TRY(st);
    for (int i = 0; i < np; ++i) HPS_CUDA(cudaEventRecord(T->gs[i].join, T->lane[2 + i].st));
  }
  // the distinct keys with their slots: compact the live slots (slot order),
  // then sort them by key (n_ws items, ~3x fewer than the occurrences) when
  // the value store is in host memory. Key order is not needed for results
  // (row sources, store lists and write-back are per key; hps_dump sorts on
  // demand), but it keeps the zero-copy store gather and write-back walking
  // host memory in address order: unsorted, e2e at c2 fell from 12.7M to
  // 8.2M ex/s, while an HBM store gains 5% without the sort.
  tile_scan(T, LiveSlot{T->tkeys[tb]}, CompactEmit{T->tkeys[tb], nullptr, l.kB, l.vB},
            Count{cap, 0}, cap_bound, &l.d->total);
  std::uint64_t* sk = l.kB;
  std::uint32_t* so = l.vB;
  if (ws_sorted(T))
    radix_sort(T, l.kB, l.vB, Count{nws, 0}, sh.own_bound, T->sort_bits, true, &sk, &so);
  const std::uint64_t wcopy = std::min(sh.own_bound, T->Wmax);  // bound, within the buffers
  HPS_CUDA(cudaMemcpyAsync(T->wsb[tb], sk, wcopy * 8, cudaMemcpyDeviceToDevice, l.st));
  HPS_CUDA(cudaMemcpyAsync(T->wsib[tb], so, wcopy * 4, cudaMemcpyDeviceToDevice, l.st));
  // rows: carry flags + table-two-back copies + the store list (HBM, full
  // grid), then the store rows (zero-copy over PCIe for a host store: a few
  // CTAs with independent loads in flight saturate the link, and leave the
  // other SMs to the running body)
  const int tp = bp.tp, tq = bp.tq;
  const std::uint64_t* pk = tp >= 0 ? T->tkeys[tp] : nullptr;
  const std::uint64_t* pc = tp >= 0 ? &T->dsc->cap[tp] : nullptr;
  const std::uint64_t* qk = tq >= 0 ? T->tkeys[tq] : nullptr;
  const std::uint64_t* qc = tq >= 0 ? &T->dsc->cap[tq] : nullptr;
  const int tq2 = bp.tq2;
  const std::uint64_t* q2k = tq2 >= 0 ? T->tkeys[tq2] : nullptr;
  const std::uint64_t* q2c = tq2 >= 0 ? &T->dsc->cap[tq2] : nullptr;
  launch(T, table_prefetch_probe_kernel, prep_grid_of(T, grid_for(sh.own_bound)), 256, 0,
         (const std::uint64_t*)T->wsb[tb], (const std::uint32_t*)T->wsib[tb],
         (const std::uint64_t*)nws, T->tvals[tb], T->csrc[tb], pk, pc, qk, qc, q2k, q2c,
         T->store != nullptr, T->store_keys, T->RW, T->need_key[tb], T->need_slot[tb],
         &T->dsc->stored_tab[tb], &T->dsc->carried_tab[tb]);
  // the store list is ready: the store gather (enqueue_store_gather, its own
  // stream, outside this graph) starts here, beside the grouping and the next
  // batch's prep — PCIe-bound on a few CTAs vs. L2-bound on the rest
  if (T->store) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(l.st, &cs);
    HPS_CUDA(cudaEventRecordWithFlags(
        T->pf_fork, l.st, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0));
  }
  if (bp.grouped)
    for (int i = 0; i < T->prep_group_lanes; ++i)
      HPS_CUDA(cudaStreamWaitEvent(l.st, T->gs[i].join, 0));
  mark(T, HPS_T_BUILD);
  return HPS_OK;
}

// Host side of a DMA transfer (cudaLaunchHostFunc, in stream order): copy
// *cnt rows between the host store and the pinned staging, split over host
// threads (the rows are random 64-512-byte records: host threads gather at
// memory speed, the PCIe link then sees one contiguous DMA).
static void CUDART_CB dma_host_rows(void* p) {
  const Tier::DmaJob& j = *static_cast<const Tier::DmaJob*>(p);
  const std::uint64_t n = *j.cnt;
  const std::size_t rb = std::size_t(j.RW) * 4;
  auto work = [&](std::uint64_t a, std::uint64_t b) {
    for (std::uint64_t i = a; i < b; ++i) {
      float* st = j.store + j.keys[i] * std::uint64_t(j.RW);
      float* sg = j.rows + i * std::uint64_t(j.RW);
      if (j.scatter) std::memcpy(st, sg, rb);
      else std::memcpy(sg, st, rb);
    }
  };
  const int T = (n < 4096 || j.threads < 2) ? 1 : j.threads;
  if (T == 1) {
    work(0, n);
    return;
  }
  std::vector<std::thread> th;
  const std::uint64_t per = (n + T - 1) / T;
  for (int t = 1; t < T; ++t)
    th.emplace_back(work, std::min(n, per * t), std::min(n, per * (t + 1)));
  work(0, std::min(n, per));
  for (auto& x : th) x.join();
}

// DMA staging of the store rows of table tb (host store, Tier::dma): the
// prep's list (keys, slots, count) to pinned memory, host threads gather the
// rows, one H2D copy, then the rows into their slots. Sizes are the shape's
// bound (known when enqueued); the count is read on both sides at run time.
static hps_status enqueue_store_gather_dma(Tier* T, const BatchShape& sh, int tb) {
  const std::uint64_t RW = std::uint64_t(T->RW);
  const std::uint64_t bound = std::min(sh.own_bound, T->Wmax);
  cudaStream_t s = T->st_pf;
  HPS_CUDA(cudaMemcpyAsync(T->g_hcnt, &T->dsc->stored_tab[tb], 8, cudaMemcpyDeviceToHost, s));
  HPS_CUDA(cudaMemcpyAsync(T->g_hkeys, T->need_key[tb], bound * 8, cudaMemcpyDeviceToHost, s));
  HPS_CUDA(cudaLaunchHostFunc(s, dma_host_rows, &T->gjob));
  HPS_CUDA(cudaMemcpyAsync(T->g_drows, T->g_hrows, bound * RW * 4, cudaMemcpyHostToDevice, s));
  const int V = vec_of(T->RW);
  auto k = V == 4 ? staged_rows_to_slots_kernel<4> : staged_rows_to_slots_kernel<1>;
  launch_on(T, s, k, grid_for(bound * (RW / V)), 256, 0, (const float*)T->g_drows,
            (const std::uint32_t*)T->need_slot[tb],
            (const unsigned long long*)&T->dsc->stored_tab[tb], T->tvals[tb], T->RW);
  return HPS_OK;
}

// The store rows of table tb (host memory over PCIe, or HBM): a streaming
// gather on st_pf, after the prep's store list; the batch's body waits for it.
static hps_status enqueue_store_gather(Tier* T, const BatchShape& sh, int tb) {
  const int E = T->RW, V = vec_of(E);  // whole rows (embedding + optimizer state)
  HPS_CUDA(cudaStreamWaitEvent(T->st_pf, T->pf_fork, 0));
  // the store rows of keys last held by the table four builds back (not a
  // proxy of this batch) arrive with its eviction write-back
  const int te = T->hist[3];
  if (te >= 0 && T->wb_pending[te]) HPS_CUDA(cudaStreamWaitEvent(T->st_pf, T->ev_wb[te], 0));
  if (T->dma) {
    HPS_TRY(enqueue_store_gather_dma(T, sh, tb));
    HPS_CUDA(cudaEventRecord(T->pf_join, T->st_pf));
    return HPS_OK;
  }
  const std::uint64_t work = sh.own_bound * std::uint64_t(E / V);
  const unsigned gg = T->store_on_host ? T->pf_ctas : grid_for(work, 256 * 4);
  const int tpb = T->store_on_host ? T->zc_threads : 256;
  auto k = V == 4 ? store_gather_kernel<4, 4> : store_gather_kernel<1, 4>;
  launch_on(T, T->st_pf, k, gg, tpb, 0, (const std::uint64_t*)T->need_key[tb],
            (const std::uint32_t*)T->need_slot[tb],
            (const unsigned long long*)&T->dsc->stored_tab[tb], (const float*)T->store,
            T->tvals[tb], E);
  HPS_CUDA(cudaEventRecord(T->pf_join, T->st_pf));
  return HPS_OK;
}

// Fused exchange (p2p.cuh p2p_send_x_kernel): mini-batch j's unique keys in
// uid order and their owner ranks into the j & 1 buffers; the owner-rank pass
// opens the next exchange round (device epoch).
static void x_keys(Tier* T, const BatchShape& sh, const BatchPlan& bp, int j) {
  const int q = j & 1;
  const std::uint64_t r0 = group_region(sh, j), ob = sh.mb_bound[j];
  launch(T, uid_keys_kernel, grid_for(ob), 256, 0, (const std::uint32_t*)(T->g_uidb[bp.tb] + r0),
         (const std::uint64_t*)T->rq_keys[bp.tb],
         (const unsigned long long*)&T->dsc->Ug[bp.tb][j], T->xukeys[q], &T->dsc->Ux[q]);
  const std::uint32_t nb =
      std::max<std::uint32_t>(1, std::uint32_t((ob + kRankTile - 1) / kRankTile));
  ++T->p2p_epoch;  // host mirror of the round the kernel opens
  launch(T, owner_rank_kernel, nb, kRankThreads, 0, (const std::uint64_t*)T->xukeys[q],
         (const std::uint64_t*)&T->dsc->Ux[q], T->G, next_lookback(T, nb), T->xorank[q],
         T->xotot[q], &T->dsc->epoch, T->dsc->xclear);
}

// One fused round: the deltas of mini-batch jd (-1: none) and the dense
// replica (dense) go to the owners with the keys of mini-batch jk (-1: none)
// in one signalled phase X; then this rank, as owner, applies every sender's
// deltas in canonical order, updates the dense weights, and serves jk's rows
// (phase Y), waiting for its own.
// Where mini-batch j's exchange keys live: the prep's pools (xprep) or the
// body's j & 1 buffers (x_keys).
struct XKeys {
  const std::uint64_t* keys = nullptr;
  const std::uint64_t* count = nullptr;
  const std::uint32_t* orank = nullptr;
  const std::uint64_t* otot = nullptr;
};
static XKeys x_src(const Tier* T, const BatchShape& sh, const BatchPlan& bp, int j) {
  XKeys x;
  if (j < 0) return x;
  if (T->xprep) {
    const std::uint64_t r0 = group_region(sh, j);
    x.keys = T->pxukeys[bp.tb] + r0;
    x.count = reinterpret_cast<const std::uint64_t*>(&T->dsc->Ug[bp.tb][j]);
    x.orank = T->pxorank[bp.tb] + r0;
    x.otot = T->pxotot[bp.tb] + std::uint64_t(j) * kMaxRanks;
  } else {
    const int q = j & 1;
    x.keys = T->xukeys[q];
    x.count = reinterpret_cast<const std::uint64_t*>(&T->dsc->Ux[q]);
    x.orank = T->xorank[q];
    x.otot = T->xotot[q];
  }
  return x;
}

static hps_status x_round(Tier* T, const BatchShape& sh, const BatchPlan& bp, int jd, bool dense,
                          int jk) {
  const int V = vec_of(T->E), G = T->G;
  const XKeys xd = x_src(T, sh, bp, jd), xk = x_src(T, sh, bp, jk);
  auto sx = V == 4 ? p2p_send_x_kernel<4> : p2p_send_x_kernel<1>;
  launch(T, sx, grid_for(T->Omax * std::uint64_t(T->E / V), 256, kSMs * 4), 256, 0, T->ctx, G,
         T->g, T->slot, T->E, xd.keys, xd.count, xd.orank, xd.otot,
         (const float*)(jd >= 0 ? T->deltas : nullptr), std::uint64_t(T->md.nw),
         (const float*)(dense ? T->dgrad : nullptr), xk.keys, xk.count, xk.orank, xk.otot,
         T->done_ctr);
  bool waited = false;
  if (jd >= 0) {  // owner apply, senders in canonical order; the first waits for X
    auto k = V == 4 ? p2p_apply_kernel<4> : p2p_apply_kernel<1>;
    for (int src : canonical_senders(T)) {
      launch(T, k, grid_for(T->slot * std::uint64_t(T->E / V), 256, kSMs * 2), 256, 0, T->ctx,
             T->g, src, T->slot, (const std::uint32_t*)T->w_rslots, T->tvals[T->cur], T->opt, G,
             waited ? -1 : int(kPhX), &T->dsc->err, 1);
      waited = true;
    }
  }
  mark(T, HPS_T_APPLY);
  if (dense) {
    launch(T, p2p_dense_update_kernel, 1, 256, 0, T->ctx, G, T->g, T->N, T->D,
           std::uint64_t(T->md.nw), T->dense, T->cfg.learning_rate, 1, (float*)nullptr,
           &T->dsc->err, waited ? -1 : int(kPhX));
    waited = true;
  }
  mark(T, HPS_T_DENSE);
  if (jk >= 0) {  // serve the next mini-batch's rows (after the apply), then wait for ours
    auto k = V == 4 ? p2p_serve_rows_kernel<4> : p2p_serve_rows_kernel<1>;
    launch(T, k, grid_for(T->Omax * std::uint64_t(T->E / V), 256, kSMs * 4), 256, 0, T->ctx, G,
           T->g, T->slot, (const std::uint64_t*)T->tkeys[T->cur], (const float*)T->tvals[T->cur],
           (const std::uint64_t*)&T->dsc->cap[T->cur], T->w_rslots, T->E, T->RW, T->done_ctr,
           &T->dsc->served, &T->dsc->err, waited ? -1 : int(kPhX), int(kPhY));
    p2p_wait(T, kPhY);
  } else if (!waited) {
    launch(T, p2p_wait_kernel, 1, 32, 0, T->ctx, G, T->g, int(kPhX), &T->dsc->err);
  }
  mark(T, HPS_T_PULL);
  return HPS_OK;
}

// The body of one batch (lane 0): carried rows from the previous table, then
// J x {shard gather, dedup, pull, fwd/bwd, sparse reduce, push + canonical
// apply, dense sync + update}. Enqueue-only (no host synchronisation, no
// host-read device values, round counter on the device), so it can be
// captured into a CUDA graph and replayed.
static hps_status enqueue_body(Tier* T, const BatchShape& sh, const BatchPlan& bp) {
  const int G = T->G, J = T->J, E = T->E;
  const std::uint64_t B = sh.B, GJ = std::uint64_t(G) * J;
  const std::int64_t* doff = T->b_off[bp.sp];
  const std::uint64_t* dkeys = T->b_keys[bp.sp];
  const std::uint8_t* dlab = T->b_lab[bp.sp];
  mark(T, -1);
  // the body's error word is this batch's from here (bodies run in order on
  // T->st; the previous one's was copied to its BatchOut already)
  zero_on(T, T->st, {{&T->dsc->err, sizeof(DevError)},
                     {&T->dsc->loss, 16},         // loss, pulled
                     {&T->dsc->fallbacks, 48}});  // fallbacks .. mid_keys
  if (bp.tp >= 0) {  // rows from the resident tables (carry-over, proxies)
    const int RW = T->RW, V = vec_of(RW);
    const unsigned gc = grid_for(sh.own_bound * std::uint64_t(RW / V));
    auto k = V == 4 ? table_carry_kernel<4> : table_carry_kernel<1>;
    launch(T, k, gc, 256, 0, (const std::uint32_t*)T->csrc[bp.tb],
           (const std::uint32_t*)T->wsib[bp.tb], (const std::uint64_t*)&T->dsc->nws_tab[bp.tb],
           (const float*)T->tvals[bp.tp], (const float*)(bp.tq >= 0 ? T->tvals[bp.tq] : nullptr),
           (const float*)(bp.tq2 >= 0 ? T->tvals[bp.tq2] : nullptr), T->tvals[bp.tb], RW);
  }
  // the mini-batches the prep did not group: grouped here on a side branch
  // (lane 3), each ready before its mini-batch and beside the previous one
  const bool side = bp.grouped && bp.prep_mbs < J;
  if (side) {
    HPS_CUDA(cudaEventRecord(T->b_fork, T->st));
    const int nl = T->body_group_lanes, b0 = T->prep_group_lanes;  // lanes after the prep's
    for (int i = 0; i < nl; ++i)
      HPS_CUDA(cudaStreamWaitEvent(T->lane[2 + b0 + i].st, T->b_fork, 0));
    hps_status gst = HPS_OK;
    for (int j = bp.prep_mbs; j < J && gst == HPS_OK; ++j) {  // alternating lanes
      const int i = (j - bp.prep_mbs) % nl;
      T->L = &T->lane[2 + b0 + i];
      gst = enqueue_grouping(T, sh, bp, T->gs[b0 + i], j, j + 1, &T->dsc->err, T->gmb_done);
    }
    T->L = &T->lane[0];
    HPS_TRY(gst);
  }
  {  // the proxies may be recycled from here on (see submit_batch)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(T->st, &cs);
    HPS_CUDA(cudaEventRecordWithFlags(T->ev_carry_sp[bp.sp], T->st,
                                      cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                          : 0));
  }
  mark(T, HPS_T_BUILD);
  // G > 1 fused exchange: the first round carries only mini-batch 0's keys
  const bool xf = G > 1 && bp.grouped && T->xfuse;
  if (xf) {
    if (T->xprep) begin_round(T, true);
    else x_keys(T, sh, bp, 0);
    mark(T, HPS_T_DEDUP);
    HPS_TRY(x_round(T, sh, bp, -1, false, 0));
  }
  // ---- mini-batches
  const int V = vec_of(E);
  for (int j = 0; j < J; ++j) {
    const std::uint64_t s = std::uint64_t(T->g) * J + j;
    const std::uint64_t n = s < B ? (B - s - 1) / GJ + 1 : 0;
    const Count on_n{&T->dsc->counts[bp.sp][j], 0};
    const std::uint64_t ob = sh.mb_bound[j];
    const ShardMap sm{s, GJ, n};
    // shard dedup (a5) + pull (a6)
    PullPlan plan;
    const std::uint32_t* occ_row = T->inv;  // occurrence -> row of `rows`
    const float* rows = T->rows;
    int rstride = E;  // the pulled rows (uid order), or the table's rows in place
    const std::int64_t* goff = nullptr;      // occurrence ids: shard-local (sort path)
    if (side && j >= bp.prep_mbs) HPS_CUDA(cudaStreamWaitEvent(T->st, T->gmb_done[j], 0));
    const std::uint64_t* Uj = &T->dsc->U;      // this mini-batch's unique keys
    const std::uint32_t* segj = T->seg;
    const std::uint32_t* exsj = T->exs;
    const std::uint32_t* slotsj = T->slots;      // uid -> table slot (G == 1)
    if (bp.grouped) {
      // grouped by slot on the prep lane (enqueue_grouping): no sort here
      const std::uint64_t r0 = group_region(sh, j);
      Uj = reinterpret_cast<const std::uint64_t*>(&T->dsc->Ug[bp.tb][j]);
      segj = T->g_segb[bp.tb] + r0 + j;
      exsj = T->g_exsb[bp.tb] + r0;
      slotsj = T->g_uidb[bp.tb] + r0;
      goff = doff;  // occurrence ids are batch key indices
      if (G == 1) {  // fwd/bwd reads the rows in place from the table
        mark(T, HPS_T_DEDUP);
        mark(T, HPS_T_PULL);
        occ_row = T->g_occslot[bp.tb];
        rows = T->tvals[T->cur];
        rstride = T->RW;
      } else if (xf) {  // rows of this mini-batch arrived in the previous round (uid order)
        Uj = x_src(T, sh, bp, j).count;
        occ_row = T->g_inv[bp.tb];
      } else {  // unique keys in uid order -> the NVLink exchange -> rows by uid
        // (the kernel also copies the count into dsc->U: no memcpy node,
        // which would break the programmatic-launch chain)
        launch(T, uid_keys_kernel, grid_for(ob), 256, 0, slotsj,
               (const std::uint64_t*)T->rq_keys[bp.tb], (const unsigned long long*)Uj,
               T->ukeys, reinterpret_cast<unsigned long long*>(&T->dsc->U));
        begin_round(T, false);
        HPS_TRY(exchange_pull(T, ob, true));
        Uj = &T->dsc->U;
        occ_row = T->g_inv[bp.tb];
      }
    } else {
      if (n) {
        tile_scan(T, ShardLen{sm, doff}, ShardLenEmit{T->occ_off, n}, Count{nullptr, n}, n,
                  &T->L->d->total);
        launch(T, shard_gather_kernel, grid_for(n * 32), 256, 0, sm, doff, dkeys,
               (const std::uint32_t*)T->occ_off, T->L->kB, T->L->vB, T->ex_of);
      }
      if (G > 1) begin_round(T, false);
      HPS_TRY(dedup_pull(T, T->L->kB, T->L->vB, on_n, ob, &plan, true, true));
    }
    // compute (a7, a8, a9); rows are in uid order (or table slots) at every G
    if (n) {
      // the big-segment plan beside fwd/bwd (st3)
      if (T->big_side) {
        HPS_CUDA(cudaEventRecord(T->fork3, T->st));
        HPS_CUDA(cudaStreamWaitEvent(T->st3, T->fork3, 0));
      }
      HPS_TRY(launch_big_plan(T, ob, Uj, segj));
      if (T->wide) {  // tcgen05 GEMMs (mlp.cuh); the weight gradients fork onto st2
        HPS_TRY(enqueue_wide(T, sm, n, goff, occ_row, rows, rstride, dlab));
      } else {
      const int LPE = E <= 8 ? 8 : (E <= 16 ? 16 : 32);
      const int epb = 128 / LPE;
      // the shared-memory row tiles of embed_sum_tiled (E == LPE, 16-B rows)
      const int tiled = T->fb_tile && E == LPE && E % 4 == 0 && rstride % 4 == 0;
      const size_t smem = size_t((T->md.nw + 1) & ~1) * 4 +
                          size_t(epb) * (T->md.hw + T->md.dw + T->md.maxw) * 8 +
                          (tiled ? 16 + size_t(epb) * 2 * kTileRows * LPE * 4 : 0);
      const unsigned blocks = unsigned(std::min<std::uint64_t>((n + epb - 1) / epb, kSMs * 8));
      // the fixed {8, 16, 1} stack over E == LPE inputs: compile-time widths
      const bool fix = T->fb_fixed && E == LPE && T->md.L == 3 && T->md.dims[0] == 8 &&
                       T->md.dims[1] == 16 && T->md.dims[2] == 1;
      auto k = LPE == 8 ? (fix ? fwd_bwd_kernel<8, true> : fwd_bwd_kernel<8>)
                        : (LPE == 16 ? (fix ? fwd_bwd_kernel<16, true> : fwd_bwd_kernel<16>)
                                     : fwd_bwd_kernel<32>);
      launch(T, k, blocks, 128, smem, T->md, sm, (const float*)T->dense,
             (const std::uint32_t*)T->occ_off, goff, occ_row, rows, rstride, dlab, T->H,
             T->DL, T->DX, &T->dsc->loss, &T->dsc->err, tiled);
      mark(T, HPS_T_FWDBWD);
      }
      if (!T->wide && T->dg_main && T->dg_fused && T->big_side) {
        // the dense gradient follows fwd/bwd on the body stream (programmatic
        // launch: no cross-branch start latency), the three sparse passes
        // fork onto st2 (short), st3 (hot keys) and st4 (medium keys)
        HPS_CUDA(cudaEventRecord(T->fork, T->st));
        HPS_CUDA(cudaStreamWaitEvent(T->st2, T->fork, 0));
        HPS_CUDA(cudaStreamWaitEvent(T->st3, T->fork, 0));
        HPS_TRY(launch_sparse_delta(T, n, plan.pos, ob, Uj, segj, exsj,
                                    bp.grouped && G == 1 ? slotsj : nullptr, true));
        launch(T, dense_grad_fused_kernel,
               dim3(dense_grad_groups(T->md), kDGFSlices / kDGFWarps), 32 * kDGFWarps, 0, T->md,
               n, (const double*)T->H, (const double*)T->DL, T->dpart, T->dg_sync, T->dgrad,
               &T->dsc->fallbacks);
        HPS_CUDA(cudaStreamWaitEvent(T->st, T->join3, 0));
        HPS_CUDA(cudaStreamWaitEvent(T->st, T->join4, 0));
        HPS_CUDA(cudaStreamWaitEvent(T->st, T->join, 0));
        mark(T, HPS_T_SPARSE);
      } else {
      if (!T->wide) {
      // dense-grad reduce on the side stream, overlapping the sparse reduce
      HPS_CUDA(cudaEventRecord(T->fork, T->st));
      HPS_CUDA(cudaStreamWaitEvent(T->st2, T->fork, 0));
      if (T->dg_fused) {
        launch_on(T, T->st2, dense_grad_fused_kernel,
                  dim3(dense_grad_groups(T->md), kDGFSlices / kDGFWarps), 32 * kDGFWarps, 0, T->md, n,
                  (const double*)T->H, (const double*)T->DL, T->dpart, T->dg_sync, T->dgrad,
                  &T->dsc->fallbacks);
      } else {
      launch_on(T, T->st2, dense_grad_p1_kernel, dim3(dense_grad_groups(T->md), kDGSlices), 32,
                0, T->md, n, (const double*)T->H, (const double*)T->DL, T->dpart);
      launch_on(T, T->st2, dense_grad_scan_kernel, unsigned((T->md.nw + 3) / 4), 128, 0, T->md,
                (const double*)T->dpart, T->dg_off, T->dg_tot);
      launch_on(T, T->st2, dense_grad_p2_kernel, dim3(dense_grad_groups(T->md), kDGSlices), 32,
                0, T->md, n, (const double*)T->H, (const double*)T->DL, T->dpart,
                (const double*)T->dg_off);
      launch_on(T, T->st2, dense_grad_fin_kernel,
                unsigned((T->md.nw + kDGFinWarps - 1) / kDGFinWarps), 32 * kDGFinWarps, 0, T->md,
                n, (const double*)T->H, (const double*)T->DL, (const double*)T->dpart,
                (const double*)T->dg_tot, T->dgrad, &T->dsc->fallbacks);
      }
      HPS_CUDA(cudaEventRecord(T->join, T->st2));
      }
      if (T->big_side) HPS_CUDA(cudaStreamWaitEvent(T->st3, T->fork, 0));  // after fwd/bwd
      HPS_TRY(launch_sparse_delta(T, n, plan.pos, ob, Uj, segj, exsj,
                                  bp.grouped && G == 1 ? slotsj : nullptr));
      mark(T, HPS_T_SPARSE);
      HPS_CUDA(cudaStreamWaitEvent(T->st, T->join, 0));
      }
    } else {
      HPS_CUDA(cudaMemsetAsync(T->dgrad, 0, std::uint64_t(T->md.nw) * 4, T->st));
    }
    mark(T, HPS_T_GRADS);
    if (xf) {  // one fused round: deltas + dense replica of j, keys of j + 1
      const bool next = j + 1 < J;
      if (next && side && j + 1 >= bp.prep_mbs)  // its grouping (and keys) on the side branch
        HPS_CUDA(cudaStreamWaitEvent(T->st, T->gmb_done[j + 1], 0));
      if (next && !T->xprep) x_keys(T, sh, bp, j + 1);
      else begin_round(T, true);
      mark(T, HPS_T_DEDUP);
      HPS_TRY(x_round(T, sh, bp, j, j != bp.skip_mb, next ? j + 1 : -1));
      continue;
    }
    // push + canonical apply (a10, a11); grouped at one rank the sparse
    // reduce already applied each key's delta in place
    if (G == 1 && bp.grouped) {
    } else if (G == 1) {
      const std::uint64_t work = ob * std::uint64_t(E / V);
      if (V == 4)
        launch(T, table_apply_kernel<4>, grid_for(work), 256, 0, slotsj,
               (const std::uint64_t*)nullptr, (const std::uint64_t*)nullptr,
               (const std::uint64_t*)nullptr, (const float*)T->deltas, Uj, std::uint64_t(0),
               T->tvals[T->cur], T->opt, &T->dsc->err);
      else
        launch(T, table_apply_kernel<1>, grid_for(work), 256, 0, slotsj,
               (const std::uint64_t*)nullptr, (const std::uint64_t*)nullptr,
               (const std::uint64_t*)nullptr, (const float*)T->deltas, Uj, std::uint64_t(0),
               T->tvals[T->cur], T->opt, &T->dsc->err);
    } else {
      HPS_TRY(push_apply(T));
    }
    mark(T, HPS_T_APPLY);
    // dense sync + update (a12), with the verification fault knob
    if (j != bp.skip_mb) HPS_TRY(dense_sync_update(T, true));
    mark(T, HPS_T_DENSE);
  }
  return HPS_OK;
}

// Write-back of table t to the value store (a13: dump_node ->
// MemPs::collect_updates, hbm_ps.hpp:224-232, mem_ps.hpp:210-245) on st_wb,
// after its body: the rows no newer resident train table holds (`newer`, up
// to 3; those hold fresher rows and write them back themselves), in key
// order. The store is exact for every key outside the resident tables, which
// is all the next builds read from it; hps_flush makes it exact for all keys.
static hps_status enqueue_writeback(Tier* T, int t, const int* newer, int n_newer) {
  const int E = T->RW, V = vec_of(E);  // whole rows (embedding + optimizer state)
  T->mirror_dirty = T->mirror != nullptr;  // the host copy is stale until the next quiesce
  HPS_CUDA(cudaStreamWaitEvent(T->st_wb, T->ev_body_tab[t], 0));
  if (T->timing) HPS_CUDA(cudaEventRecord(T->ev_wbt[t][0], T->st_wb));
  const std::uint64_t* nk[3] = {nullptr, nullptr, nullptr};
  const std::uint64_t* nc[3] = {nullptr, nullptr, nullptr};
  for (int i = 0; i < n_newer && i < 3; ++i) {
    nk[i] = T->tkeys[newer[i]];
    nc[i] = &T->dsc->cap[newer[i]];
  }
  HPS_CUDA(cudaMemsetAsync(&T->dsc->wb_n[t], 0, 8, T->st_wb));
  launch_on(T, T->st_wb, table_evict_filter_kernel, prep_grid_of(T, grid_for(T->Wmax)), 256, 0,
            (const std::uint64_t*)T->wsb[t], (const std::uint32_t*)T->wsib[t],
            (const std::uint64_t*)&T->dsc->nws_tab[t], nk[0], nc[0], nk[1], nc[1], nk[2], nc[2],
            T->store_keys, T->wb_key[t], T->wb_slot[t], &T->dsc->wb_n[t], &T->dsc->wb_total);
  const std::uint64_t work = T->Wmax * std::uint64_t(E / V);
  if (T->dma) {  // rows compacted on the device, one D2H copy, host threads scatter
    auto kc = V == 4 ? slots_to_staged_rows_kernel<4> : slots_to_staged_rows_kernel<1>;
    launch_on(T, T->st_wb, kc, grid_for(work), 256, 0, (const std::uint32_t*)T->wb_slot[t],
              (const unsigned long long*)&T->dsc->wb_n[t], (const float*)T->tvals[t], T->w_drows,
              E);
    HPS_CUDA(cudaMemcpyAsync(T->w_hcnt, &T->dsc->wb_n[t], 8, cudaMemcpyDeviceToHost, T->st_wb));
    HPS_CUDA(cudaMemcpyAsync(T->w_hkeys, T->wb_key[t], T->Wmax * 8, cudaMemcpyDeviceToHost,
                             T->st_wb));
    HPS_CUDA(cudaMemcpyAsync(T->w_hrows, T->w_drows, T->Wmax * std::uint64_t(E) * 4,
                             cudaMemcpyDeviceToHost, T->st_wb));
    HPS_CUDA(cudaLaunchHostFunc(T->st_wb, dma_host_rows, &T->wjob));
    if (T->timing) HPS_CUDA(cudaEventRecord(T->ev_wbt[t][1], T->st_wb));
    HPS_CUDA(cudaEventRecord(T->ev_wb[t], T->st_wb));
    T->wb_pending[t] = true;
    T->wb_timed[t] = T->timing;
    return HPS_OK;
  }
  // posted PCIe writes: a few CTAs saturate the link without holding SMs
  const unsigned gw = T->store_on_host ? T->wb_ctas : grid_for(work, 256 * 4);
  const int tpb = T->store_on_host ? T->zc_threads : 256;
  auto k = V == 4 ? store_scatter_kernel<4, 4> : store_scatter_kernel<1, 4>;
  launch_on(T, T->st_wb, k, gw, tpb, 0, (const std::uint64_t*)T->wb_key[t],
            (const std::uint32_t*)T->wb_slot[t], (const unsigned long long*)&T->dsc->wb_n[t],
            (const float*)T->tvals[t], T->store, E, T->mirror_pages);
  if (T->timing) HPS_CUDA(cudaEventRecord(T->ev_wbt[t][1], T->st_wb));
  HPS_CUDA(cudaEventRecord(T->ev_wb[t], T->st_wb));
  T->wb_pending[t] = true;
  T->wb_timed[t] = T->timing;
  return HPS_OK;
}

// Train tables of the current store newer than table t (newest first).
static int newer_tables(const Tier* T, int t, int* out) {
  int n = 0;
  for (int q = 0; q < kTables; ++q)
    if (q != t && T->tab_wb[q] && T->tab_age[q] > T->tab_age[t]) out[n++] = q;
  std::sort(out, out + n, [T](int a, int b) { return T->tab_age[a] > T->tab_age[b]; });
  return std::min(n, 3);
}

// Every resident train table's rows that are not in the store yet, oldest
// first (enqueue-only on st_wb): afterwards the store holds every trained row.
static hps_status flush_all(Tier* T) {
  if (!T->store) return HPS_OK;
  int order[kTables], n = 0;
  for (int q = 0; q < kTables; ++q)
    if (T->tab_wb[q] && !T->tab_flushed[q]) order[n++] = q;
  std::sort(order, order + n, [T](int a, int b) { return T->tab_age[a] < T->tab_age[b]; });
  for (int i = 0; i < n; ++i) {
    int newer[kTables];
    const int nn = newer_tables(T, order[i], newer);
    HPS_TRY(enqueue_writeback(T, order[i], newer, nn));
    T->tab_flushed[order[i]] = true;
  }
  return HPS_OK;
}

// Fold a finished write-back's duration into the WRITEBACK timing slot.
static void wb_account(Tier* T, int p, bool wait) {
  if (!T->wb_timed[p]) return;
  if (wait) cudaEventSynchronize(T->ev_wbt[p][1]);
  else if (cudaEventQuery(T->ev_wbt[p][1]) != cudaSuccess) return;
  float ms = 0;
  cudaEventElapsedTime(&ms, T->ev_wbt[p][0], T->ev_wbt[p][1]);
  T->acc_ms[HPS_T_WRITEBACK] += ms;
  T->wb_timed[p] = false;
}

// Order stream s after the pending write-backs (of table p, or all: -1).
static hps_status wb_fence(Tier* T, int p = -1, cudaStream_t s = nullptr) {
  for (int q = 0; q < kTables; ++q) {
    if ((p >= 0 && q != p) || !T->wb_pending[q]) continue;
    HPS_CUDA(cudaStreamWaitEvent(s ? s : T->st, T->ev_wb[q], 0));
  }
  return HPS_OK;
}

// Capture `enqueue` on the current lane's stream once per key (no launch):
// a whole prep or body becomes one graph. The cache keeps the 256 most
// recently used graphs; an evicted one may still be running (batches are in
// flight), so it is destroyed only at the next quiesce.
// HPS_PROG_EDGES=1: in a captured body graph, the edges from fwd/bwd to the
// reduces that other streams run after it (dense gradient, medium and
// hot-key segments) become programmatic edges, as the same-stream launches
// already are: those kernels may launch as fwd/bwd's blocks retire and wait
// for its results in griddepcontrol.wait (pdl_wait, their first statement),
// instead of paying a cross-stream launch after its completion.
static bool is_fwd_bwd(const void* f) {
  return f == reinterpret_cast<const void*>(fwd_bwd_kernel<8>) ||
         f == reinterpret_cast<const void*>(fwd_bwd_kernel<16>) ||
         f == reinterpret_cast<const void*>(fwd_bwd_kernel<32>) ||
         f == reinterpret_cast<const void*>(fwd_bwd_kernel<8, true>) ||
         f == reinterpret_cast<const void*>(fwd_bwd_kernel<16, true>);
}
static bool is_side_reduce(const void* f) {
  return f == reinterpret_cast<const void*>(dense_grad_fused_kernel) ||
         f == reinterpret_cast<const void*>(big_fused_kernel) ||
         f == reinterpret_cast<const void*>(sparse_mid_cert_kernel<4>) ||
         f == reinterpret_cast<const void*>(sparse_mid_cert_kernel<8>) ||
         f == reinterpret_cast<const void*>(sparse_mid_cert_kernel<16>) ||
         f == reinterpret_cast<const void*>(sparse_mid_cert_kernel<32>);
}
static const void* kernel_of(cudaGraphNode_t n) {
  cudaGraphNodeType ty;
  if (cudaGraphNodeGetType(n, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) return nullptr;
  cudaKernelNodeParams p{};
  if (cudaGraphKernelNodeGetParams(n, &p) != cudaSuccess) return nullptr;
  return p.func;
}
static hps_status programmatic_side_edges(cudaGraph_t g, bool all, bool join_edges,
                                          bool any_into_side) {
  std::size_t ne = 0;
  HPS_CUDA(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne));
  if (!ne) return HPS_OK;
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  std::vector<cudaGraphEdgeData> ed(ne);
  HPS_CUDA(cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne));
  for (std::size_t i = 0; i < ne; ++i) {
    if (ed[i].type != cudaGraphDependencyTypeDefault) continue;
    const void* kf = kernel_of(from[i]);
    const void* kt = kernel_of(to[i]);
    if (!kf || !kt) continue;  // memset / copy / event nodes keep full edges
    // all: every kernel -> kernel edge (every kernel here opens with pdl_wait,
    // and a programmatic port fires only once all of the upstream kernel's
    // blocks have exited, so no early block can starve it of SMs)
    // mode 4: every kernel edge into a side reduce (also big_plan -> medium keys)
    const bool side_in = (is_fwd_bwd(kf) || any_into_side) && is_side_reduce(kt);
    // mode 3 adds the joins: the side reduces -> the dense update after them
    const bool side_out = join_edges && is_side_reduce(kf) &&
                          kt == reinterpret_cast<const void*>(dense_update_kernel);
    if (!all && !side_in && !side_out) continue;
    HPS_CUDA(cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &ed[i], 1));
    cudaGraphEdgeData pe{};
    pe.from_port = cudaGraphKernelNodePortProgrammatic;
    pe.type = cudaGraphDependencyTypeProgrammatic;
    HPS_CUDA(cudaGraphAddDependencies_v2(g, &from[i], &to[i], &pe, 1));
  }
  return HPS_OK;
}

template <class Fn>
static hps_status capture_graph(Tier* T, const std::vector<std::uint64_t>& key, Fn&& enqueue,
                                GraphEntry** out) {
  cudaStream_t s = T->L->st;
  auto it = T->graphs.find(key);
  if (it == T->graphs.end()) {
    if (T->graphs.size() >= 256) {  // bounded cache: evict the least recently used
      auto lru = T->graphs.begin();
      for (auto i = T->graphs.begin(); i != T->graphs.end(); ++i)
        if (i->second.last_use < lru->second.last_use) lru = i;
      T->retired.push_back(lru->second.exec);
      T->graphs.erase(lru);
    }
    GraphEntry ge;
    const std::uint64_t l0 = T->launches, e0 = T->p2p_epoch;
    const std::size_t ev0 = T->ev_phase.size();
    HPS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const hps_status st = enqueue();
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st != HPS_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ce != cudaSuccess)
      return set_error(HPS_ERR_CUDA, "cuda: graph capture: %s", cudaGetErrorString(ce));
    if (T->prog_edges)
      HPS_TRY(programmatic_side_edges(g, T->prog_edges == 2, T->prog_edges == 3,
                                      T->prog_edges == 4));
    // node priorities follow the capturing stream (body high, prep low)
    const cudaError_t ie =
        cudaGraphInstantiate(&ge.exec, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess)
      return set_error(HPS_ERR_CUDA, "cuda: graph instantiate: %s", cudaGetErrorString(ie));
    ge.launches = T->launches - l0;
    ge.epochs = T->p2p_epoch - e0;
    ge.ev_phase.assign(T->ev_phase.begin() + ev0, T->ev_phase.end());
    ge.ev_lane.assign(T->ev_lane.begin() + ev0, T->ev_lane.end());
    T->launches = l0;  // counted per replay
    T->p2p_epoch = e0;
    T->ev_phase.resize(ev0);
    T->ev_lane.resize(ev0);
    ++T->graph_captures;
    it = T->graphs.emplace(key, std::move(ge)).first;
  }
  it->second.last_use = ++T->graph_clock;
  *out = &it->second;
  return HPS_OK;
}

// Capture once per key, then replay.
template <class Fn>
static hps_status run_graph(Tier* T, const std::vector<std::uint64_t>& key, Fn&& enqueue) {
  GraphEntry* ge = nullptr;
  HPS_TRY(capture_graph(T, key, std::forward<Fn>(enqueue), &ge));
  HPS_CUDA(cudaGraphLaunch(ge->exec, T->L->st));
  T->launches += ge->launches;
  T->p2p_epoch += ge->epochs;
  T->ev_phase.insert(T->ev_phase.end(), ge->ev_phase.begin(), ge->ev_phase.end());
  T->ev_lane.insert(T->ev_lane.end(), ge->ev_lane.begin(), ge->ev_lane.end());
  return HPS_OK;
}

// ------------------------------------------------------ the batch pipeline

// Wait for the oldest in-flight batch and park its result in T->done.
static void complete_oldest(Tier* T) {
  const BatchPlan bp = T->inflight.front();
  T->inflight.pop_front();
  Tier::Done d{bp.id, HPS_OK, std::string(), hps_batch_stats{}};
  const cudaError_t ce = cudaEventSynchronize(T->ev_body_sp[bp.sp]);
  if (ce != cudaSuccess) {
    d.st = set_error(HPS_ERR_CUDA, "cuda: %s", cudaGetErrorString(ce));
    d.msg = error_message();
  } else {
    const BatchOut& o = T->hout[bp.sp];
    const int G = T->G, J = T->J;
    const std::uint64_t GJ = std::uint64_t(G) * J;
    hps_batch_stats& st = d.stats;
    st.loss_sum = o.loss;
    std::uint64_t ex = 0;
    for (int j = 0; j < J; ++j) {
      const std::uint64_t sh = std::uint64_t(T->g) * J + j;
      ex += sh < bp.B ? (bp.B - sh - 1) / GJ + 1 : 0;
    }
    st.examples = ex;
    st.working_set = o.n_ws;
    st.table_capacity = o.cap;
    st.pulled_keys = o.pulled;
    st.carried_rows = o.carried;
    st.store_rows = o.stored;
    T->rows_read += o.stored;
    st.exact_fallbacks = o.fallbacks;
    st.served_keys = o.served;
    st.big_segments = o.big_keys;
    st.max_segment_chunks = o.max_chunks;
    st.big_occurrences = o.big_occ;
    st.mid_segments = o.mid_keys;
    st.occurrences = bp.occ_total;
    // first failing stage: the key-range check, the build, the body
    const DevError& e = o.err_stage.code ? o.err_stage : (o.err_prep.code ? o.err_prep : o.err);
    if (e.code) {
      d.st = device_error_status(T, e, "device table: missing key ");
      d.msg = error_message();
    }
  }
  if (T->timing) timing_end(T);
  for (int q = 0; q < kTables; ++q) wb_account(T, q, false);
  if (T->trace) {  // never waits: the write-back shown is batch id-3's, if done
    float v[8] = {}, gv[2] = {};
    for (int k = 0; k < 6; ++k) cudaEventElapsedTime(&v[k], T->tr_base, T->tr[bp.sp][k]);
    if (T->store)
      for (int k = 0; k < 2; ++k) cudaEventElapsedTime(&gv[k], T->tr_base, T->trg[bp.sp][k]);
    const int w = int((bp.id + 1) & 3);  // (id - 3) mod 4
    if (T->store && bp.id >= 3 && cudaEventQuery(T->trw[w][1]) == cudaSuccess) {
      cudaEventElapsedTime(&v[6], T->tr_base, T->trw[w][0]);
      cudaEventElapsedTime(&v[7], T->tr_base, T->trw[w][1]);
    }
    std::fprintf(stderr,
                 "[trace] batch %llu: stage %.3f-%.3f prep %.3f-%.3f gather %.3f-%.3f "
                 "body %.3f-%.3f | wb(batch-3) %.3f-%.3f\n",
                 (unsigned long long)bp.id, v[0], v[1], v[2], v[3], gv[0], gv[1], v[4], v[5], v[6],
                 v[7]);
  }
  T->done.push_back(std::move(d));
}

// Every in-flight batch done; the main stream ordered after the write-backs.
// The parity API (build / pull / push / drain / dump ...) starts from here.
static hps_status quiesce(Tier* T) {
  if (!T->inflight.empty()) {
    while (!T->inflight.empty()) complete_oldest(T);
    // the batches reported their own errors; the parity API starts clean
    HPS_CUDA(cudaMemsetAsync(&T->dsc->err, 0, sizeof(DevError), T->st));
  }
  if (!T->retired.empty()) {  // no batch in flight: evicted graphs can go
    HPS_CUDA(cudaStreamSynchronize(T->st));
    for (cudaGraphExec_t g : T->retired) cudaGraphExecDestroy(g);
    T->retired.clear();
  }
  HPS_TRY(flush_all(T));
  HPS_TRY(wb_fence(T));
  if (T->mirror && T->mirror_dirty) {  // the host store is observed: make it exact
    // (the pages written back since the last copy, in runs of DMA copies)
    const std::uint64_t np = T->mirror_hpages.size();
    const std::uint64_t prow = std::uint64_t(1) << kMirrorPageShift;
    const std::uint64_t rowb = std::uint64_t(T->RW) * 4;
    HPS_CUDA(cudaStreamSynchronize(T->st_wb));
    if (T->G > 1) {  // this rank's rows only, zero-copy writes (the array may be shared)
      const int rw4 = T->RW / 4;
      const std::uint64_t keys = T->mirror_bytes / rowb;
      launch_on(T, T->st_wb, mirror_owned_copyback_kernel, kSMs * 4, 512, 0,
                reinterpret_cast<const float4*>(T->mirror),
                reinterpret_cast<float4*>(T->mirror_hmapped),
                (const std::uint8_t*)T->mirror_pages, keys, rw4, T->G, T->g);
      T->mirror_d2h += keys / std::uint64_t(T->G) * rowb;  // (at most)
      HPS_CUDA(cudaMemsetAsync(T->mirror_pages, 0, np, T->st_wb));
      HPS_CUDA(cudaStreamSynchronize(T->st_wb));
      T->mirror_dirty = false;
      return HPS_OK;
    }
    HPS_CUDA(cudaMemcpy(T->mirror_hpages.data(), T->mirror_pages, np, cudaMemcpyDeviceToHost));
    for (std::uint64_t p = 0; p < np;) {
      if (!T->mirror_hpages[p]) {
        ++p;
        continue;
      }
      std::uint64_t q = p;
      while (q < np && T->mirror_hpages[q]) ++q;
      const std::uint64_t off = p * prow * rowb;
      const std::uint64_t len = std::min(q * prow * rowb, T->mirror_bytes) - off;
      HPS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(T->mirror_host) + off,
                               reinterpret_cast<const char*>(T->mirror) + off, len,
                               cudaMemcpyDeviceToHost, T->st_wb));
      T->mirror_d2h += len;
      p = q;
    }
    HPS_CUDA(cudaMemsetAsync(T->mirror_pages, 0, np, T->st_wb));
    HPS_CUDA(cudaStreamSynchronize(T->st_wb));
    T->mirror_dirty = false;
  }
  return HPS_OK;
}

// Graph keys of a batch's prep and body: the shape plus the table / staging
// rotation they are captured for.
static std::vector<std::uint64_t> prep_key(const Tier* T, const BatchShape& sh,
                                           const BatchPlan& bp) {
  return {1, sh.B, sh.own_bound, sh.batch_bound, std::uint64_t(bp.tb), std::uint64_t(bp.tp + 1),
          std::uint64_t(bp.tq + 1), std::uint64_t(bp.tq2 + 1), std::uint64_t(bp.sp),
          std::uint64_t(bp.prep_mbs), reinterpret_cast<std::uint64_t>(T->store), T->store_keys,
          std::uint64_t(T->store_on_host), std::uint64_t(T->timing)};
}
static std::vector<std::uint64_t> body_key(const Tier* T, const BatchShape& sh,
                                           const BatchPlan& bp) {
  std::vector<std::uint64_t> key = {2, sh.B, sh.own_bound, std::uint64_t(bp.tb),
                                    std::uint64_t(bp.tp + 1), std::uint64_t(bp.tq + 1),
                                    std::uint64_t(bp.tq2 + 1), std::uint64_t(bp.sp),
                                    std::uint64_t(bp.prep_mbs), std::uint64_t(T->timing)};
  for (int j = 0; j < T->J; ++j) key.push_back(sh.mb_bound[j]);
  return key;
}

// Steady state of the rotation: every table role is filled, so the next
// batches of this shape differ only by the rotation offset.
static bool steady(const Tier* T, const BatchPlan& bp) {
  return bp.tp >= 0 && (!T->store || (bp.tq >= 0 && bp.tq2 >= 0));
}

// The same batch one to kTables-1 rotation steps later (tables and staging
// slots advance together).
static BatchPlan rotated(const BatchPlan& bp, int r) {
  BatchPlan q = bp;
  auto rot = [r](int x) { return x < 0 ? -1 : (x + r) % kTables; };
  q.tb = rot(bp.tb);
  q.tp = rot(bp.tp);
  q.tq = rot(bp.tq);
  q.tq2 = rot(bp.tq2);
  q.sp = (bp.sp + r) % kSlots;
  return q;
}

// The first steady batch of a shape captures the prep (body) graphs of all
// kTables rotations at once, so the batches that follow never pay a capture
// and instantiate (five warm-ups reached 2 of the 5 rotations,
// leaving three captures inside the timed region). Capture only: nothing is
// launched; the lanes' host look-back state is reset per capture (captured
// launches bake context-relative tickets) and restored.
static hps_status precapture_rotations(Tier* T, const BatchShape& sh, const BatchPlan& bp,
                                       bool body) {
  // body: lane 0 + its grouping lanes; prep: lane 1 + its grouping lanes
  int lanes[1 + kGroupLanes];
  int nl = 0;
  lanes[nl++] = body ? 0 : 1;
  const int g0 = body ? 2 + T->prep_group_lanes : 2;
  const int gn = body ? T->body_group_lanes : T->prep_group_lanes;
  for (int i = 0; i < gn; ++i) lanes[nl++] = g0 + i;
  std::uint64_t tk[1 + kGroupLanes];
  std::uint32_t lb[1 + kGroupLanes];
  for (int i = 0; i < nl; ++i) {
    tk[i] = T->lane[lanes[i]].tickets;
    lb[i] = T->lane[lanes[i]].lb_local;
  }
  const int cur = T->cur;
  hps_status st = HPS_OK;
  for (int r = 1; r < kTables && st == HPS_OK; ++r) {
    const BatchPlan q = rotated(bp, r);
    for (int i = 0; i < nl; ++i) {
      T->lane[lanes[i]].tickets = tk[i];
      T->lane[lanes[i]].lb_local = lb[i];
    }
    GraphEntry* ge = nullptr;
    if (body) {
      T->cur = q.tb;
      st = capture_graph(T, body_key(T, sh, q), [&] { return enqueue_body(T, sh, q); }, &ge);
    } else {
      st = capture_graph(T, prep_key(T, sh, q), [&] { return enqueue_prep(T, sh, q); }, &ge);
    }
  }
  T->cur = cur;
  for (int i = 0; i < nl; ++i) {
    T->lane[lanes[i]].tickets = tk[i];
    T->lane[lanes[i]].lb_local = lb[i];
  }
  return st;
}

// Stage (H2D + counts + range check, st_stage) -> prep (lane 1) -> body
// (lane 0) -> write-back (st_wb) of one batch, all enqueued; the host blocks
// only on the stage's count round-trip. At most kSlots batches are in flight.
static hps_status submit_batch(Tier* T, std::uint64_t B, const std::int64_t* offsets,
                               const std::uint64_t* keys, const std::uint8_t* labels,
                               int on_device, std::uint64_t* id_out) {
  if (T->N != 1) return set_error(HPS_ERR_ARG, "train_batch: one node per box (nodes must be 1)");
  if (B > T->Bmax)
    return set_error(HPS_ERR_CAPACITY, "train_batch: %llu examples exceed max_batch_examples",
                     (unsigned long long)B);
  if (T->timing)  // phases are attributed without overlap: one batch at a time
    while (!T->inflight.empty()) complete_oldest(T);
  while (T->inflight.size() >= std::size_t(kMaxInflight)) complete_oldest(T);
  const int G = T->G, J = T->J;
  BatchPlan bp;
  bp.id = T->submitted;
  bp.B = B;
  bp.sp = int(T->submitted % kSlots);
  bp.tb = next_table(T);
  bp.tp = T->cur;
  bp.tq = (T->store && T->prev >= 0 && T->prev != bp.tb && T->tab_wb[T->prev]) ? T->prev : -1;
  bp.tq2 = (bp.tq >= 0 && T->prev2 >= 0 && T->prev2 != bp.tb && T->tab_wb[T->prev2])
               ? T->prev2 : -1;
  bp.step = T->step;
  const int sp = bp.sp;
  // ---- stage into the tier's own buffers (captured graphs never see caller
  // pointers), after the body that last used this staging slot
  cudaStream_t ss = T->st_stage;
  timing_begin(T);
  mark_stage(T, -1);
  if (T->sp_pending[sp]) HPS_CUDA(cudaStreamWaitEvent(ss, T->ev_body_sp[sp], 0));
  if (T->trace) cudaEventRecord(T->tr[sp][0], ss);
  std::uint64_t O = 0;
  if (on_device) {
    HPS_CUDA(cudaMemcpyAsync(T->b_off[sp], offsets, (B + 1) * 8, cudaMemcpyDeviceToDevice, ss));
    HPS_CUDA(cudaMemcpyAsync(&T->hsc->total_unused, offsets + B, 8, cudaMemcpyDeviceToHost, ss));
    HPS_CUDA(cudaStreamSynchronize(ss));
    O = std::uint64_t(T->hsc->total_unused);
    if (O > T->Omax)
      return set_error(HPS_ERR_CAPACITY, "train_batch: %llu keys exceed max_batch_keys",
                       (unsigned long long)O);
    HPS_CUDA(cudaMemcpyAsync(T->b_keys[sp], keys, O * 8, cudaMemcpyDeviceToDevice, ss));
    HPS_CUDA(cudaMemcpyAsync(T->b_lab[sp], labels, B, cudaMemcpyDeviceToDevice, ss));
  } else {
    O = std::uint64_t(offsets[B]);
    if (O > T->Omax)
      return set_error(HPS_ERR_CAPACITY, "train_batch: %llu keys exceed max_batch_keys",
                       (unsigned long long)O);
    HPS_CUDA(cudaMemcpyAsync(T->b_off[sp], offsets, (B + 1) * 8, cudaMemcpyHostToDevice, ss));
    HPS_CUDA(cudaMemcpyAsync(T->b_keys[sp], keys, O * 8, cudaMemcpyHostToDevice, ss));
    HPS_CUDA(cudaMemcpyAsync(T->b_lab[sp], labels, B, cudaMemcpyHostToDevice, ss));
  }
  zero_on(T, ss, {{T->dsc->counts[sp], sizeof(T->dsc->counts[sp])},
                  {&T->dsc->serr[sp], sizeof(DevError)}});
  launch_on(T, ss, batch_count_kernel, kSMs * 4, 256, 0, (const std::int64_t*)T->b_off[sp],
            (const std::uint64_t*)T->b_keys[sp], B, G, T->g, J,
            T->cfg.key_space ? T->cfg.key_space : ~std::uint64_t(0), T->dsc->counts[sp],
            &T->dsc->serr[sp]);
  // Host batch at one rank: the shape counts follow from the offsets alone
  // (per-shard occurrences; every key is owned), so the host does not wait
  // for the copy — the device counts and the key-range check (its error is
  // reported by hps_wait_batch) follow in stream order. Otherwise one
  // round-trip (and at G > 1 the collective error agreement).
  const bool host_counts = !on_device && G == 1;
  if (host_counts) {
    std::uint64_t* hc = T->hsc->counts[sp];
    for (int i = 0; i < 66; ++i) hc[i] = 0;
    for (std::uint64_t i = 0; i < B; ++i) hc[i % J] += std::uint64_t(offsets[i + 1] - offsets[i]);
    hc[J] = O;
    hc[J + 1] = O;
    mark_stage(T, HPS_T_STAGE);
    if (T->trace) cudaEventRecord(T->tr[sp][1], ss);
    HPS_CUDA(cudaEventRecord(T->ev_staged, ss));
  } else {
    HPS_CUDA(cudaMemcpyAsync(T->hsc->counts[sp], T->dsc->counts[sp],
                             sizeof(T->dsc->counts[sp]), cudaMemcpyDeviceToHost, ss));
    mark_stage(T, HPS_T_STAGE);
    if (T->trace) cudaEventRecord(T->tr[sp][1], ss);
    HPS_CUDA(cudaEventRecord(T->ev_staged, ss));
    HPS_TRY(check_device_error(T, "device table: missing key ", true, ss, &T->dsc->serr[sp]));
  }
  for (int j = 0; j < J; ++j) bp.occ_total += T->hsc->counts[sp][j];
  const std::uint64_t own = T->hsc->counts[sp][J];
  if (own > T->Wmax || bp.occ_total > T->Omax)
    return set_error(HPS_ERR_CAPACITY, "train_batch: batch exceeds configured maxima");
  // ---- shape: power-of-two upper bounds of the counts, so one captured
  // graph serves every batch of a shape
  BatchShape sh;
  sh.B = B;
  sh.own_bound = shape_bound(own);
  sh.batch_bound = shape_bound(std::uint64_t(T->hsc->counts[sp][J + 1]));
  for (int j = 0; j < J; ++j) sh.mb_bound[j] = shape_bound(T->hsc->counts[sp][j]);
  const std::int64_t first_mb = T->step * J;
  if (T->cfg.inject_skip_sync >= first_mb && T->cfg.inject_skip_sync < first_mb + J)
    bp.skip_mb = int(T->cfg.inject_skip_sync - first_mb);
  {  // slot grouping (G == 1) when its shared-memory bitmaps fit
    const std::uint64_t nmax = (B + std::uint64_t(G) * J - 1) / (std::uint64_t(G) * J);
    const std::size_t words = std::size_t((nmax + 31) / 32);
    bp.grouped = T->hash_dedup &&
                 std::size_t(kGroupSortThreads / 32) * 8 * words <= kGroupSmemMax;
    // who groups what: with a host store the prep is short next to the PCIe
    // traffic and takes every mini-batch; with an HBM store the body takes
    // the later half beside its compute (c2: 0.80 vs 0.85 ms/step; with a host
    // store 1.36 vs 1.49). At G > 1 the exchange waits leave the body's
    // SMs idle enough that the prep takes every mini-batch too (c2: +1.6%
    // at N = 2, +2.1% at N = 4)
    bp.prep_mbs = T->prep_mbs > 0 ? std::min(T->prep_mbs, J)
                                  : (T->store_on_host || T->G > 1 ? J : std::max(1, J / 2));
  }
  // ---- prep on lane 1, beside the previous body
  {
    cudaStream_t ps = T->lane[1].st;
    HPS_CUDA(cudaStreamWaitEvent(ps, T->ev_staged, 0));
    // (the proxies' rows are copied by this batch's body, after theirs); the
    // batch two back read the table this build recycles as its oldest proxy
    if (bp.id >= 2) {
      const int sp2 = int((bp.id - 2) % kSlots);
      HPS_CUDA(cudaStreamWaitEvent(ps, T->ev_carry_sp[sp2], 0));
    }
    // HPS_PREP_LAG=1: the build also waits for the previous body's carry, so
    // it does not crowd that body's start (the batch boundary)
    if (T->prep_lag1 && bp.id >= 1)
      HPS_CUDA(cudaStreamWaitEvent(ps, T->ev_carry_sp[(bp.id - 1) % kSlots], 0));
    if (T->body_pending[bp.tb]) HPS_CUDA(cudaStreamWaitEvent(ps, T->ev_body_tab[bp.tb], 0));
    if (T->wb_pending[bp.tb]) HPS_CUDA(cudaStreamWaitEvent(ps, T->ev_wb[bp.tb], 0));
    if (T->trace) cudaEventRecord(T->tr[sp][2], ps);
    if (bp.grouped) {  // the prep grouping lanes' look-back contexts: after the
      // previous prep (whose graph ran their last groupings), before this one
      for (int i = 0; i < T->prep_group_lanes; ++i) {
        Lane& ln = T->lane[2 + i];
        HPS_CUDA(cudaStreamWaitEvent(ln.st, T->ev_prep, 0));
        T->L = &ln;
        open_lookback_context(T);
        HPS_CUDA(cudaEventRecord(T->gs[i].ctx, ln.st));
        HPS_CUDA(cudaStreamWaitEvent(ps, T->gs[i].ctx, 0));
      }
    }
    T->L = &T->lane[1];
    open_lookback_context(T);
    hps_status st;
    if (T->use_graphs) {
      const std::vector<std::uint64_t> key = prep_key(T, sh, bp);
      st = HPS_OK;
      if (steady(T, bp) && !T->graphs.count(key)) st = precapture_rotations(T, sh, bp, false);
      if (st == HPS_OK) st = run_graph(T, key, [&] { return enqueue_prep(T, sh, bp); });
    } else {
      st = enqueue_prep(T, sh, bp);
    }
    T->L = &T->lane[0];
    HPS_TRY(st);
    HPS_CUDA(cudaEventRecord(T->ev_prep, ps));
    if (T->trace) cudaEventRecord(T->tr[sp][3], ps);
    if (T->store) {
      if (T->trace) {
        HPS_CUDA(cudaStreamWaitEvent(T->st_pf, T->pf_fork, 0));
        cudaEventRecord(T->trg[sp][0], T->st_pf);
      }
      HPS_TRY(enqueue_store_gather(T, sh, bp.tb));
      if (T->trace) cudaEventRecord(T->trg[sp][1], T->st_pf);
    }
  }
  // ---- body on lane 0 (after its prep and its store rows)
  HPS_CUDA(cudaStreamWaitEvent(T->st, T->ev_prep, 0));
  if (T->store) HPS_CUDA(cudaStreamWaitEvent(T->st, T->pf_join, 0));
  if (bp.grouped && bp.prep_mbs < J) {  // the look-back contexts of lanes 3, 4 (the
    // body's grouping branches): after the previous body, before this one
    for (int i = 0; i < T->body_group_lanes; ++i) {
      Lane& lx = T->lane[2 + T->prep_group_lanes + i];
      if (bp.id >= 1)
        HPS_CUDA(cudaStreamWaitEvent(lx.st, T->ev_body_sp[(bp.id - 1) % kSlots], 0));
      T->L = &lx;
      open_lookback_context(T);
      T->L = &T->lane[0];
      HPS_CUDA(cudaEventRecord(T->gs[T->prep_group_lanes + i].ctx, lx.st));
      HPS_CUDA(cudaStreamWaitEvent(T->st, T->gs[T->prep_group_lanes + i].ctx, 0));
    }
  }
  if (T->trace) cudaEventRecord(T->tr[sp][4], T->st);
  open_lookback_context(T);
  T->prev2 = T->prev;
  T->prev = bp.tp;
  T->cur = bp.tb;
  T->ws = T->wsb[bp.tb];
  T->ws_idx = T->wsib[bp.tb];
  T->ws_sorted = ws_sorted(T);
  if (T->use_graphs && bp.skip_mb < 0) {
    const std::vector<std::uint64_t> key = body_key(T, sh, bp);
    if (steady(T, bp) && !T->graphs.count(key)) HPS_TRY(precapture_rotations(T, sh, bp, true));
    HPS_TRY(run_graph(T, key, [&] { return enqueue_body(T, sh, bp); }));
  } else {
    HPS_TRY(enqueue_body(T, sh, bp));
  }
  BatchOut* ho = &T->hout[sp];
  const int tb = bp.tb;
  launch(T, batch_out_kernel, 1, 32, 0, (const Scalars*)T->dsc, tb, sp, ho);
  if (T->trace) cudaEventRecord(T->tr[sp][5], T->st);
  HPS_CUDA(cudaEventRecord(T->ev_body_tab[tb], T->st));
  HPS_CUDA(cudaEventRecord(T->ev_body_sp[sp], T->st));
  T->body_pending[tb] = true;
  T->sp_pending[sp] = true;
  T->tab_wb[tb] = T->store != nullptr;
  T->tab_flushed[tb] = false;
  T->tab_age[tb] = ++T->builds;
  for (int k = kTables - 1; k > 0; --k) T->hist[k] = T->hist[k - 1];
  T->hist[0] = tb;
  // ---- eviction write-back (the collect stage) on st_wb, overlapping the
  // next batches: the next batch reads its rows from the tables of this and
  // the two previous batches, and the store — so the table three builds back
  // gives up its rows now (those no newer table holds), and the next batch's
  // store gather waits for it
  const int tr = T->hist[3];
  if (tr >= 0 && T->store && T->tab_wb[tr] && !T->tab_flushed[tr]) {
    int newer[kTables];
    const int nn = newer_tables(T, tr, newer);
    HPS_CUDA(cudaStreamWaitEvent(T->st_wb, T->ev_prep, 0));  // this batch's keys are final
    if (T->trace) cudaEventRecord(T->trw[bp.id & 3][0], T->st_wb);
    HPS_TRY(enqueue_writeback(T, tr, newer, nn));
    if (T->trace) cudaEventRecord(T->trw[bp.id & 3][1], T->st_wb);
    T->tab_flushed[tr] = true;
  }
  T->inflight.push_back(bp);
  ++T->submitted;
  ++T->step;
  if (id_out) *id_out = bp.id;
  return HPS_OK;
}

}  // namespace hpsgpu

// =================================================================== ABI

using namespace hpsgpu;

struct hps_tier : public hpsgpu::Tier {};

bool hpsgpu::pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("HPS_PDL");
    return !v || std::atoi(v) != 0;
  }();
  return on;
}

bool hpsgpu::debug_sync_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("HPS_DEBUG_SYNC");
    return v && std::atoi(v) != 0;
  }();
  return on;
}

extern "C" {

const char* hps_last_error(void) { return error_message(); }
const char* hps_version(void) { return "hps-b200 0.1 (sm_100a)"; }

hps_status hps_get_unique_id(uint8_t id[HPS_NCCL_ID_BYTES]) {
  if (!id) return set_error(HPS_ERR_ARG, "null id");
  if (!nccl().ok) return set_error(HPS_ERR_NCCL, "nccl: %s", nccl().why.c_str());
  ncclUniqueId u;
  HPS_NCCL(nccl().GetUniqueId(&u));
  std::memcpy(id, &u, HPS_NCCL_ID_BYTES);
  return HPS_OK;
}

static bool is_pow2(std::uint64_t x) { return x && !(x & (x - 1)); }

hps_status hps_create(const hps_config* cfg, const uint8_t* nccl_id, hps_tier_t* out) {
  if (!cfg || !out) return set_error(HPS_ERR_ARG, "null argument");
  *out = nullptr;
  const hps_config& c = *cfg;
  if (c.nodes < 1 || !is_pow2(std::uint64_t(c.nodes)))
    return set_error(HPS_ERR_ARG, "topology: num_nodes must be a power of two");
  if (c.devices_per_node < 1 || !is_pow2(std::uint64_t(c.devices_per_node)))
    return set_error(HPS_ERR_ARG, "topology: devices_per_node must be a power of two");
  const int G = c.nodes * c.devices_per_node;
  if (c.rank < 0 || c.rank >= G) return set_error(HPS_ERR_ARG, "rank out of range");
  if (G > 256) return set_error(HPS_ERR_ARG, "at most 256 devices");
  if (c.embedding_dim < 1) return set_error(HPS_ERR_ARG, "config: embedding_dim > 0");
  if (c.num_layers < 1 || c.num_layers > HPS_MAX_LAYERS || c.layer_dims[c.num_layers - 1] != 1)
    return set_error(HPS_ERR_ARG, "config: layer_dims must end in 1");
  if (c.minibatches < 1 || c.minibatches > 64)
    return set_error(HPS_ERR_ARG, "config: minibatches_per_batch in [1, 64]");
  if (!(c.learning_rate > 0.0f))
    return set_error(HPS_ERR_ARG, "config: learning_rate must be positive");
  if (c.max_batch_keys >= (1ull << 31) || c.max_batch_examples >= (1ull << 31))
    return set_error(HPS_ERR_ARG, "batch maxima must be < 2^31");
  // layers up to kMaxHidden wide run the exact f64 fwd_bwd_kernel; a wider
  // hidden layer (or HPS_WIDE=1) selects the tcgen05 GEMM path (mlp.cuh)
  bool wide = false;
  {
    const char* v = std::getenv("HPS_WIDE");
    wide = v && std::atoi(v) != 0;
  }
  for (int l = 0; l < c.num_layers; ++l) {
    if (c.layer_dims[l] < 1 || c.layer_dims[l] > 4096)
      return set_error(HPS_ERR_ARG, "layer width must be in [1, 4096]");
    if (c.layer_dims[l] > std::uint64_t(kMaxHidden)) wide = true;
  }
  if (wide && c.num_layers < 2)
    return set_error(HPS_ERR_ARG, "the wide MLP path needs a hidden layer");
  if (c.embedding_dim > 256) return set_error(HPS_ERR_ARG, "embedding_dim <= 256");
  if (c.optimizer != HPS_OPT_SGD && c.optimizer != HPS_OPT_ADAGRAD)
    return set_error(HPS_ERR_ARG, "config: optimizer must be HPS_OPT_SGD or HPS_OPT_ADAGRAD");
  if (c.optimizer == HPS_OPT_ADAGRAD && !(c.adagrad_eps > 0.0f))
    return set_error(HPS_ERR_ARG, "config: adagrad_eps must be positive");
  if (G > 1 && !nccl_id) return set_error(HPS_ERR_ARG, "nccl_id required when N*D > 1");
  if (G > 1 && !nccl().ok) return set_error(HPS_ERR_NCCL, "nccl: %s", nccl().why.c_str());

  auto* t = new hps_tier();
  t->cfg = c;
  t->N = c.nodes;
  t->D = c.devices_per_node;
  t->G = G;
  t->g = c.rank;
  t->E = c.embedding_dim;
  t->J = c.minibatches;
  t->wide = wide;
  if (const char* v = std::getenv("HPS_TF32_1X")) t->gemm_split3 = std::atoi(v) == 0;
  t->RW = c.optimizer == HPS_OPT_ADAGRAD ? 2 * t->E : t->E;
  t->opt = Optim{c.optimizer, t->E, t->RW, c.learning_rate, c.adagrad_eps};
  t->Bmax = std::max<std::uint64_t>(c.max_batch_examples, 1);
  t->Omax = std::max<std::uint64_t>(c.max_batch_keys, 1);
  t->Wmax = c.max_working_set ? c.max_working_set : t->Omax;
  t->Wmax = std::max(t->Wmax, t->Omax);
  t->capmax = table_capacity(t->Wmax);
  if (const char* v = std::getenv("HPS_PF_CTAS")) t->pf_ctas = unsigned(std::max(1, std::atoi(v)));
  if (const char* v = std::getenv("HPS_WB_CTAS")) t->wb_ctas = unsigned(std::max(1, std::atoi(v)));
  if (const char* v = std::getenv("HPS_TRACE")) t->trace = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_DEDUP")) t->hash_dedup = std::strcmp(v, "sort") != 0;
  if (const char* v = std::getenv("HPS_GRAPHS")) t->use_graphs = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_PREP_GROUP"))
    t->prep_mbs = std::max(0, std::atoi(v));
  if (const char* v = std::getenv("HPS_PRIO")) t->priorities = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_BIG_SIDE")) t->big_side = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_FB_TILE")) t->fb_tile = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_DG_FUSED")) t->dg_fused = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_MID_CERT")) t->mid_cert = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_PREP_GRID")) t->prep_grid = unsigned(std::max(0, std::atoi(v)));
  if (const char* v = std::getenv("HPS_GROUP_PRIO")) t->group_prio = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_GROUP_FUSED")) t->group_fused = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_TAIL_PRIO")) t->tail_prio = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_DG_MAIN")) t->dg_main = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_PREP_LAG")) t->prep_lag1 = std::atoi(v) == 1;
  if (const char* v = std::getenv("HPS_PROG_EDGES")) t->prog_edges = std::atoi(v);
  if (const char* v = std::getenv("HPS_SHORT_GRID")) t->short_grid = unsigned(std::max(0, std::atoi(v)));
  if (const char* v = std::getenv("HPS_FB_FIXED")) t->fb_fixed = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_STORE_MIRROR_GB")) t->mirror_gb = std::atof(v);
  if (const char* v = std::getenv("HPS_PREP_GROUP_LANES"))
    t->prep_group_lanes = std::min(kGroupLanes - 1, std::max(1, std::atoi(v)));
  if (const char* v = std::getenv("HPS_BODY_GROUP_LANES"))
    t->body_group_lanes = std::min(kGroupLanes - t->prep_group_lanes, std::max(1, std::atoi(v)));
  if (const char* v = std::getenv("HPS_SHORT_DPT")) {
    const int d = std::atoi(v);
    if (d == 1 || (d == 4 && c.embedding_dim % 4 == 0) || (d == 8 && c.embedding_dim % 8 == 0))
      t->short_dpt = d;
  }
  if (const char* v = std::getenv("HPS_MID_SEG"))
    t->mid_max = std::uint32_t(std::min(kMidMaxSeg, std::max(kLongSeg, std::atoi(v))));
  if (const char* v = std::getenv("HPS_SHORT_SEG"))
    t->short_max = std::uint32_t(std::min(kLongSeg, std::max(1, std::atoi(v))));
  if (const char* v = std::getenv("HPS_FOLD_WAIT")) t->fold_wait = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_XFUSE")) t->xfuse = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_XPREP")) t->xprep = std::atoi(v) != 0;
  if (const char* v = std::getenv("HPS_STAGE"))
    t->stage_mode = std::strcmp(v, "dma") == 0 ? 1 : (std::strcmp(v, "zc") == 0 ? 0 : -1);
  if (const char* v = std::getenv("HPS_WS_SORT")) t->ws_sort = std::atoi(v) != 0 ? 1 : 0;
  if (const char* v = std::getenv("HPS_ZC_THREADS")) t->zc_threads = std::max(32, std::atoi(v));
  t->nmb_max = t->Bmax;  // a shard never exceeds the batch
  t->nshard = (t->Bmax + std::uint64_t(G) * t->cfg.minibatches - 1) /
              (std::uint64_t(G) * t->cfg.minibatches);
  {
    int bits = 64;
    if (c.key_space) {
      bits = 0;
      while (bits < 64 && (std::uint64_t(1) << bits) < c.key_space) ++bits;
    }
    t->sort_bits = std::max(bits, 1);
  }
  // model dims
  {
    ModelDims& m = t->md;
    m.E = t->E;
    m.L = c.num_layers;
    int off = 0, in = t->E, hw = 0, dw = 0, maxw = t->E;
    for (int l = 0; l < m.L; ++l) {
      m.dims[l] = int(c.layer_dims[l]);
      m.ins[l] = in;
      m.offs[l] = off;
      m.hoff[l] = hw;
      m.doff[l] = dw;
      hw += in;
      dw += m.dims[l];
      off += (in + 1) * m.dims[l];
      in = m.dims[l];
      maxw = std::max(maxw, m.dims[l]);
    }
    m.nw = off;
    m.hw = hw;
    m.dw = dw;
    m.maxw = maxw;
    // the order-free embed_sum bound (model.cuh embed_sum_exact): 29 is the
    // exactness limit; HPS_EMBED_SLACK may only tighten it (tests use it to
    // force the in-order fallback for part of a batch)
    m.exact_slack = 29;
    if (const char* v = std::getenv("HPS_EMBED_SLACK"))
      m.exact_slack = std::max(-1, std::min(29, std::atoi(v)));
  }

  auto fail = [&](hps_status s) {
    hps_destroy(t);
    return s;
  };
  cudaError_t e = cudaSetDevice(c.cuda_device);
  if (e != cudaSuccess)
    return fail(set_error(HPS_ERR_CUDA, "cuda: cudaSetDevice(%d): %s", c.cuda_device,
                          cudaGetErrorString(e)));
  {  // test knob: every certified sum takes its exact fallback (model.cuh)
    const char* v = std::getenv("HPS_CERT_FORCE_FAIL");
    const int force = v ? std::atoi(v) != 0 : 0;
    e = cudaMemcpyToSymbol(g_cert_force_fail, &force, sizeof(int));
    if (e != cudaSuccess)
      return fail(set_error(HPS_ERR_CUDA, "cuda: %s", cudaGetErrorString(e)));
  }
  {
    auto ev = [&](cudaEvent_t* x, bool timed) {
      if (e == cudaSuccess)
        e = timed ? cudaEventCreate(x) : cudaEventCreateWithFlags(x, cudaEventDisableTiming);
    };
    // the body (critical path) outranks the work that overlaps it
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (!t->priorities) lo = hi = 0;
    auto str = [&](cudaStream_t* x, int prio) {
      if (e == cudaSuccess) e = cudaStreamCreateWithPriority(x, cudaStreamNonBlocking, prio);
    };
    // within the body, the long-latency reductions (medium keys on st4, hot
    // keys on st3) outrank the short-key pass and the dense gradient, whose
    // many CTAs would otherwise take every slot first and start them late
    // (HPS_TAIL_PRIO=0: all four equal)
    const int body2 = (t->tail_prio && hi < lo) ? hi + 1 : hi;
    str(&t->st, body2);
    str(&t->st2, body2);
    str(&t->st3, hi);
    str(&t->st4, hi);
    str(&t->lane[1].st, lo);
    // lane 2 groups the next batch (prep, low); lane 3 groups this body's
    // later mini-batches, which wait for it — at prep priority too: body
    // priority (HPS_GROUP_PRIO=1) measured 28.9M vs 30.0M ex/s on c2 (its
    // kernels then crowd the running mini-batch's reduce instead)
    for (int i = 0; i < kGroupLanes; ++i)
      str(&t->lane[2 + i].st, (t->group_prio && i >= t->prep_group_lanes) ? hi : lo);
    str(&t->st_stage, lo);
    str(&t->st_wb, lo);
    str(&t->st_pf, lo);
    ev(&t->fork, false);
    ev(&t->join, false);
    ev(&t->fork3, false);
    ev(&t->join3, false);
    ev(&t->fork4, false);
    ev(&t->join4, false);
    ev(&t->ev_staged, false);
    ev(&t->ev_prep, false);
    ev(&t->pf_fork, false);
    ev(&t->g_fork, false);
    ev(&t->b_fork, false);
    for (auto& x : t->gmb_done) ev(&x, false);
    for (GroupState& g : t->gs) {
      ev(&g.join, false);
      ev(&g.ctx, false);
    }
    ev(&t->pf_join, false);
    for (int i = 0; i < kTables; ++i) {
      ev(&t->ev_body_tab[i], false);
      ev(&t->ev_wb[i], false);
      ev(&t->ev_wbt[i][0], true);
      ev(&t->ev_wbt[i][1], true);
    }
    for (auto& x : t->ev_body_sp) ev(&x, false);
    for (auto& x : t->ev_carry_sp) ev(&x, false);
    if (t->trace) {
      ev(&t->tr_base, true);
      for (auto& row : t->tr)
        for (auto& x : row) ev(&x, true);
      for (auto& row : t->trw)
        for (auto& x : row) ev(&x, true);
      for (auto& row : t->trg)
        for (auto& x : row) ev(&x, true);
      if (e == cudaSuccess) e = cudaEventRecord(t->tr_base, t->st);
    }
    t->lane[0].st = t->st;
    if (e != cudaSuccess)
      return fail(set_error(HPS_ERR_CUDA, "cuda: stream: %s", cudaGetErrorString(e)));
  }

  {
    // dynamic shared memory of the model kernels (per-example scratch, streamed records)
    const int big = 200 * 1024;
    const size_t need_grad = 0;
    const size_t need_fwd = size_t((t->md.nw + 1) & ~1) * 4 +
                            size_t(16) * (t->md.hw + t->md.dw + t->md.maxw) * 8;
    if (!t->wide && (need_grad > size_t(big) || need_fwd > size_t(big)))
      return fail(set_error(HPS_ERR_ARG, "dense model too large for the fused kernels"));

    cudaFuncSetAttribute(fwd_bwd_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(fwd_bwd_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(fwd_bwd_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(fwd_bwd_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(fwd_bwd_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(sparse_mid_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(mid_smem(1)));
    cudaFuncSetAttribute(sparse_mid_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(mid_smem(2)));
    cudaFuncSetAttribute(sparse_mid_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(mid_smem(4)));
    cudaFuncSetAttribute(umma_gemm_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(gemm_smem(128, true)));
    cudaFuncSetAttribute(umma_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(gemm_smem(64, true)));
    cudaFuncSetAttribute(umma_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(gemm_smem(32, true)));
    cudaFuncSetAttribute(group_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kGroupSmemMax));
    cudaFuncSetAttribute(group_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kGroupSmemMax));
    cudaFuncSetAttribute(group_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kGroupSmemMax));
  }
  const std::uint64_t O = t->Omax, W = t->Wmax, E = std::uint64_t(t->E);
  hps_status s = HPS_OK;
#define A(ptr, n) \
  if ((s = dalloc(t, &t->ptr, (n))) != HPS_OK) return fail(s)
  A(dsc, 1);
  if ((e = cudaMallocHost(&t->hsc, sizeof(Scalars))) != cudaSuccess)
    return fail(set_error(HPS_ERR_CUDA, "cuda: host alloc: %s", cudaGetErrorString(e)));
  if ((e = cudaMallocHost(&t->hout, kSlots * sizeof(BatchOut))) != cudaSuccess)
    return fail(set_error(HPS_ERR_CUDA, "cuda: host alloc: %s", cudaGetErrorString(e)));
  for (int i = 0; i < kTables; ++i) {
    A(tkeys[i], t->capmax);
    A(tvals[i], t->capmax * std::uint64_t(t->RW));
    A(wsb[i], W);
    A(wsib[i], W);
    A(csrc[i], W);
  }
  for (int i = 0; i < kTables; ++i) {
    A(need_key[i], W);
    A(need_slot[i], W);
    A(wb_key[i], W);
    A(wb_slot[i], W);
  }
  // per-slot grouping arrays cover the largest slot space: the batch table
  // (G == 1) or the request table (G > 1)
  t->rq_cap = 1;
  while (t->rq_cap < 2 * std::max(O, W)) t->rq_cap <<= 1;
  t->gslots = G > 1 ? std::max(t->capmax, t->rq_cap) : t->capmax;
  for (GroupState& g : t->gs) {
    if ((s = dalloc(t, &g.gcnt, t->gslots)) != HPS_OK ||
        (s = dalloc(t, &g.slot_uid, t->gslots)) != HPS_OK)
      return fail(s);
  }
  t->ws = t->wsb[0];
  t->ws_idx = t->wsib[0];
  const std::uint64_t S = std::max(O, W);
  const std::uint64_t status_words =
      std::max<std::uint64_t>(std::uint64_t(kDigits) * sort_tiles(S), scan_tiles(S)) + 1;
  for (int li = 0; li < 2 + kGroupLanes; ++li) {
    Lane& l = t->lane[li];
    if (li < 2 &&  // the grouping lanes only scan: no radix scratch
        ((s = dalloc(t, &l.kA, S)) != HPS_OK || (s = dalloc(t, &l.kB, S)) != HPS_OK ||
         (s = dalloc(t, &l.vA, S)) != HPS_OK || (s = dalloc(t, &l.vB, S)) != HPS_OK ||
         (s = dalloc(t, &l.ghist, std::uint64_t(kMaxPasses) * kDigits)) != HPS_OK))
      return fail(s);
    if ((s = dalloc(t, &l.status, status_words)) != HPS_OK ||
        (s = dalloc(t, &l.ticket, 1)) != HPS_OK || (s = dalloc(t, &l.d, 1)) != HPS_OK)
      return fail(s);
    l.status_words = status_words;
    cudaMemsetAsync(l.ticket, 0, 8, t->st);
    cudaMemsetAsync(l.status, 0, status_words * 8, t->st);
    cudaMemsetAsync(l.d, 0, sizeof(LaneDev), t->st);
  }
  for (int i = 0; i < kSlots; ++i) {
    A(b_off[i], t->Bmax + 1);
    A(b_keys[i], O);
    A(b_lab[i], t->Bmax);
  }
  A(occ_off, t->nmb_max + 1);
  A(ex_of, S);
  A(inv, S);
  A(seg, S + 1);
  A(uidv, S);
  A(pos, S);
  A(slots, S);
  A(exs, S);
  A(orank, S);
  t->g_pool = 2 * S + std::uint64_t(t->J) * 4096 + 64;  // >= the sum of the shape bounds
  for (int i = 0; i < kTables; ++i) {
    A(g_occslot[i], S);
    if (G > 1) {
      A(g_inv[i], S);
      A(rq_keys[i], t->rq_cap);
    }
    A(g_segb[i], t->g_pool + 64);
    A(g_exsb[i], t->g_pool);
    A(g_uidb[i], t->g_pool);
    if (G > 1) {
      A(pxukeys[i], t->g_pool);
      A(pxorank[i], t->g_pool);
      A(pxotot[i], std::uint64_t(64) * kMaxRanks);
    }
  }
  for (int i = 0; i < kTables; ++i) {
    A(g_tick[i], S);
    A(g_segocc[i], t->g_pool);
    A(g_exof[i], S);
  }
  for (GroupState& g : t->gs) {
    if ((s = dalloc(t, &g.g_long, S)) != HPS_OK || (s = dalloc(t, &g.g_huge, S)) != HPS_OK ||
        (s = dalloc(t, &g.g_dup, S)) != HPS_OK || (s = dalloc(t, &g.gn, 4)) != HPS_OK)
      return fail(s);
  }
  t->part_cap = S;  // a partition can never overflow
  for (GroupState& g : t->gs) {
    if ((s = dalloc(t, &g.part_slot, std::uint64_t(kGroupParts) * S)) != HPS_OK ||
        (s = dalloc(t, &g.part_n, std::uint64_t(kGroupParts) * kGroupPartStride)) != HPS_OK ||
        (s = dalloc(t, &g.part_base, kGroupParts)) != HPS_OK)
      return fail(s);
  }
  A(otot, kMaxRanks);
  A(big_list, S / (kLongSeg + 1) + 2);
  A(mid_list, S / 2 + 2);  // keys longer than short_max >= 1
  A(chunk_off, S / (kLongSeg + 1) + 3);
  A(key_done, S / (kLongSeg + 1) + 2);
  // fused big-segment items: one per (key, chunk of fuse_chunk(E) occurrences)
  t->fuse_items = S / std::uint64_t(fuse_chunk(int(E))) + S / (kLongSeg + 1) + 2;
  A(chunk_tot, t->fuse_items * E);
  A(item_key, t->fuse_items);
  A(item_chunk, t->fuse_items);
  A(fuse_ticket, 1);
  A(ukeys, S);
  if (G > 1)
    for (int q = 0; q < 2; ++q) {
      A(xukeys[q], S);
      A(xorank[q], S);
      A(xotot[q], kMaxRanks);
    }
  if (G == 1) A(rows, S * E);  // G > 1: inside the exported window (peers write it)
  A(deltas, S * E);
  A(hstage, S * E);
  if (!t->wide) {  // the exact path's per-example records
    A(H, t->nmb_max * std::uint64_t(t->md.hw) + 2);   // +2: 16-B rounded bulk copies
    A(DL, t->nmb_max * std::uint64_t(t->md.dw) + 2);
  } else {
    const std::uint64_t ns = t->nshard;
    A(wX, ns * E);
    std::uint64_t pmax = std::uint64_t(kSMs) * kGemmBM * 256;
    for (int l = 0; l + 1 < t->md.L; ++l) {
      A(wH[l], ns * std::uint64_t(t->md.dims[l]));
      A(wdZ[l], ns * std::uint64_t(t->md.dims[l]));
      pmax = std::max(pmax, std::uint64_t(t->md.dims[l]) * (t->md.ins[l] + 1));
    }
    A(wdz, ns);
    A(wP, pmax);
    t->wP_cap = pmax;
  }
  A(DX, t->nmb_max * E);
  if (!t->wide) {  // the certified dense-gradient reduce of the exact path
    A(dpart, std::uint64_t(t->md.nw) * std::max(kDGSlices, kDGFSlices) * 4);
    A(dg_off, std::uint64_t(t->md.nw) * kDGSlices);
    A(dg_tot, std::uint64_t(t->md.nw) * 4);
    A(dg_sync, dense_grad_groups(t->md));
  }
  A(dense, t->md.nw);
  A(dgrad, t->md.nw);
#undef A
  for (GroupState& g : t->gs) {
    cudaMemsetAsync(g.gcnt, 0, t->gslots * 4, t->st);
    cudaMemsetAsync(g.part_n, 0, std::uint64_t(kGroupParts) * kGroupPartStride * 4, t->st);
  }
  cudaMemsetAsync(t->key_done, 0, (S / (kLongSeg + 1) + 2) * 4, t->st);
  if (t->dg_sync) cudaMemsetAsync(t->dg_sync, 0, dense_grad_groups(t->md) * 4, t->st);
  if ((e = cudaMemsetAsync(t->dsc, 0, sizeof(Scalars), t->st)) != cudaSuccess)
    return fail(set_error(HPS_ERR_CUDA, "cuda: memset: %s", cudaGetErrorString(e)));
  t->hsc->rq_capv = t->rq_cap;
  cudaMemcpyAsync(&t->dsc->rq_capv, &t->hsc->rq_capv, 8, cudaMemcpyHostToDevice, t->st);
  // replicate_dense(init_dense(cfg)) — the init stream is host-side std::mt19937_64
  {
    std::vector<float> w(t->md.nw);
    init_dense_host(&c, w.data(), w.size());
    if ((e = cudaMemcpy(t->dense, w.data(), w.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(set_error(HPS_ERR_CUDA, "cuda: %s", cudaGetErrorString(e)));
  }
  if (G > 1) {
    ncclUniqueId u;
    std::memcpy(&u, nccl_id, HPS_NCCL_ID_BYTES);
    ncclResult_t r = nccl().CommInitRank(&t->comm, G, u, t->g);
    if (r != ncclSuccess)
      return fail(set_error(HPS_ERR_NCCL, "nccl: init: %s", nccl().GetErrorString(r)));
    if ((s = setup_p2p(t, S)) != HPS_OK) return fail(s);
  }
  if ((e = cudaStreamSynchronize(t->st)) != cudaSuccess)
    return fail(set_error(HPS_ERR_CUDA, "cuda: %s", cudaGetErrorString(e)));
  *out = t;
  return HPS_OK;
}

hps_status hps_destroy(hps_tier_t t) {
  if (!t) return HPS_OK;
  cudaSetDevice(t->cfg.cuda_device);
  if (t->dsc) quiesce(t);  // in-flight batches, then every resident row to the store
  for (cudaStream_t x :
       {t->st, t->lane[1].st, t->st_stage, t->st_wb, t->st2, t->st3, t->st4, t->st_pf})
    if (x) cudaStreamSynchronize(x);
  for (int gl = 0; gl < kGroupLanes; ++gl)
    if (t->lane[2 + gl].st) cudaStreamSynchronize(t->lane[2 + gl].st);
  if (t->comm) nccl().CommDestroy(t->comm);
  if (t->mirror) cudaFree(t->mirror);
  if (t->mirror_pages) cudaFree(t->mirror_pages);
  if (t->mirror_registered) cudaHostUnregister(t->mirror_host);
  cudaFree(t->pend_keys);
  cudaFree(t->pend_deltas);
  for (auto& kv : t->graphs) cudaGraphExecDestroy(kv.second.exec);
  for (cudaGraphExec_t g : t->retired) cudaGraphExecDestroy(g);
  for (void* p : t->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : t->allocs) cudaFree(p);
  if (t->hsc) cudaFreeHost(t->hsc);
  if (t->hout) cudaFreeHost(t->hout);
  if (t->store_registered) cudaHostUnregister(t->store_host);
  for (void* p : t->pinned) cudaFreeHost(p);
  for (auto& ev : t->evpool) cudaEventDestroy(ev);
  if (t->fork) cudaEventDestroy(t->fork);
  if (t->join) cudaEventDestroy(t->join);
  if (t->fork3) cudaEventDestroy(t->fork3);
  if (t->join3) cudaEventDestroy(t->join3);
  if (t->fork4) cudaEventDestroy(t->fork4);
  if (t->join4) cudaEventDestroy(t->join4);
  for (int p = 0; p < kTables; ++p) {
    for (cudaEvent_t x : {t->ev_wb[p], t->ev_body_tab[p], t->ev_wbt[p][0], t->ev_wbt[p][1]})
      if (x) cudaEventDestroy(x);
  }
  for (cudaEvent_t x : t->ev_body_sp)
    if (x) cudaEventDestroy(x);
  for (cudaEvent_t x : t->ev_carry_sp)
    if (x) cudaEventDestroy(x);
  for (cudaEvent_t x : {t->ev_staged, t->ev_prep, t->pf_fork, t->pf_join, t->g_fork, t->b_fork})
    if (x) cudaEventDestroy(x);
  for (cudaEvent_t x : t->gmb_done)
    if (x) cudaEventDestroy(x);
  for (GroupState& g : t->gs)
    for (cudaEvent_t x : {g.join, g.ctx})
      if (x) cudaEventDestroy(x);
  for (cudaStream_t x : {t->lane[1].st, t->st_stage, t->st_wb, t->st_pf})
    if (x) cudaStreamDestroy(x);
  for (int gl = 0; gl < kGroupLanes; ++gl)
    if (t->lane[2 + gl].st) cudaStreamDestroy(t->lane[2 + gl].st);
  if (t->st2) cudaStreamDestroy(t->st2);
  if (t->st3) cudaStreamDestroy(t->st3);
  if (t->st4) cudaStreamDestroy(t->st4);
  if (t->st) cudaStreamDestroy(t->st);
  delete t;
  return HPS_OK;
}

#define HPS_ENTER(t)                                         \
  if (!(t)) return set_error(HPS_ERR_ARG, "null handle");    \
  HPS_CUDA(cudaSetDevice((t)->cfg.cuda_device))

// The parity API runs after every in-flight batch (and its write-back).
#define HPS_ENTER_Q(t) \
  HPS_ENTER(t);        \
  HPS_TRY(quiesce(t))

// The growable staging scratch (HostValue rows of hps_build, hps_dump's
// rows), at least `floats` floats.
static hps_status ensure_staged(Tier* t, std::uint64_t floats) {
  if (t->staged_cap >= floats) return HPS_OK;
  HPS_CUDA(cudaStreamSynchronize(t->st));
  if (t->staged) cudaFree(t->staged);
  t->staged = nullptr;
  t->staged_cap = 0;
  HPS_CUDA(cudaMalloc(&t->staged, floats * 4));
  t->staged_cap = floats;
  return HPS_OK;
}

static hps_status build_impl(Tier* t, const uint64_t* keys, uint64_t n, const float* host_rows,
                             bool owned_only) {
  if (n > t->Wmax)
    return set_error(HPS_ERR_CAPACITY, "build: %llu keys exceed max_working_set %llu",
                     (unsigned long long)n, (unsigned long long)t->Wmax);
  if (n && !keys) return set_error(HPS_ERR_ARG, "null keys");
  if (n) {
    HPS_CUDA(cudaMemcpyAsync(t->lane[0].kB, keys, n * 8, cudaMemcpyHostToDevice, t->st));
    launch(t, iota_kernel, grid_for(n), 256, 0, t->lane[0].vB, n);
  }
  {
    const int nxt = next_table(t);
    t->ws = t->wsb[nxt];
    t->ws_idx = t->wsib[nxt];
  }
  const float* staged = nullptr;
  if (host_rows && n) {
    HPS_TRY(ensure_staged(t, n * std::uint64_t(t->RW)));
    HPS_CUDA(cudaMemcpyAsync(t->staged, host_rows, n * std::uint64_t(t->RW) * 4,
                             cudaMemcpyHostToDevice, t->st));
    staged = t->staged;
  }
  std::uint64_t* sk = nullptr;
  std::uint32_t* so = nullptr;
  open_lookback_context(t);
  if (n) {
    radix_sort(t, t->lane[0].kB, t->lane[0].vB, Count{nullptr, n}, n, 64, true, &sk, &so);
    // owned_only: keep key % G == g; otherwise every given key (the caller
    // placed them, e.g. a range-split policy)
    const std::uint64_t G = owned_only ? std::uint64_t(t->G) : 1;
    const std::uint64_t g = owned_only ? std::uint64_t(t->g) : 0;
    tile_scan(t, RunStartOwned{sk, G, g},
              CompactEmit{sk, so, t->ws, t->ws_idx}, Count{nullptr, n}, n, &t->dsc->n_ws);
  } else {
    HPS_CUDA(cudaMemsetAsync(&t->dsc->n_ws, 0, 8, t->st));
  }
  build_table(t, n, t->ws_idx, staged);
  t->ws_sorted = true;
  return check_device_error(t, "device table: missing key ");
}

hps_status hps_build(hps_tier_t t, const uint64_t* keys, uint64_t n, const float* host_rows) {
  HPS_ENTER_Q(t);
  return build_impl(t, keys, n, host_rows, true);
}

hps_status hps_build_placed(hps_tier_t t, const uint64_t* keys, uint64_t n,
                            const float* host_rows) {
  HPS_ENTER_Q(t);
  return build_impl(t, keys, n, host_rows, false);
}

static hps_status require_built(Tier* t) {
  if (t->cur < 0) return set_error(HPS_ERR_NOT_BUILT, "hbm: tables not built");
  return HPS_OK;
}

hps_status hps_pull(hps_tier_t t, const uint64_t* keys, uint64_t n, float* out_rows) {
  HPS_ENTER_Q(t);
  HPS_TRY(require_built(t));
  if (n > t->Omax)
    return set_error(HPS_ERR_CAPACITY, "pull: %llu keys exceed max_batch_keys",
                     (unsigned long long)n);
  if (n) {
    HPS_CUDA(cudaMemcpyAsync(t->lane[0].kB, keys, n * 8, cudaMemcpyHostToDevice, t->st));
    launch(t, iota_kernel, grid_for(n), 256, 0, t->lane[0].vB, n);
  }
  PullPlan plan;
  open_lookback_context(t);
  if (t->G > 1) begin_round(t, false);
  HPS_TRY(dedup_pull(t, t->lane[0].kB, t->lane[0].vB, Count{nullptr, n}, n, &plan, true));
  HPS_TRY(check_device_error(t, "device table: missing key ", true));
  if (n) {
    launch(t, scatter_rows_kernel, grid_for(n * t->E), 256, 0, (const std::uint32_t*)t->inv,
           plan.pos, n, t->E, (const float*)t->rows, t->deltas);
    HPS_CUDA(cudaMemcpyAsync(out_rows, t->deltas, n * std::uint64_t(t->E) * 4,
                             cudaMemcpyDeviceToHost, t->st));
  }
  HPS_CUDA(cudaStreamSynchronize(t->st));
  return HPS_OK;
}

hps_status hps_push(hps_tier_t t, const uint64_t* keys, const float* deltas, uint64_t n) {
  HPS_ENTER_Q(t);
  HPS_TRY(require_built(t));
  if (n > t->Omax)
    return set_error(HPS_ERR_CAPACITY, "push: %llu keys exceed max_batch_keys",
                     (unsigned long long)n);
  if (n) {
    HPS_CUDA(cudaMemcpyAsync(t->lane[0].kB, keys, n * 8, cudaMemcpyHostToDevice, t->st));
    HPS_CUDA(cudaMemcpyAsync(t->hstage, deltas, n * std::uint64_t(t->E) * 4,
                             cudaMemcpyHostToDevice, t->st));
    launch(t, iota_kernel, grid_for(n), 256, 0, t->lane[0].vB, n);
  }
  PullPlan plan;
  open_lookback_context(t);
  if (t->G > 1) begin_round(t, false);
  HPS_TRY(dedup_pull(t, t->lane[0].kB, t->lane[0].vB, Count{nullptr, n}, n, &plan, false));
  HPS_CUDA(cudaMemcpyAsync(&t->hsc->U, &t->dsc->U, 8, cudaMemcpyDeviceToHost, t->st));
  HPS_CUDA(cudaStreamSynchronize(t->st));
  // a duplicate key is reported only after the collective completes, so no
  // rank is left waiting on a peer that bailed out
  const bool dup = t->hsc->U != n;
  if (n)  // deltas into send order (uid order when G == 1)
    launch(t, permute_rows_kernel, grid_for(n * t->E), 256, 0, (const std::uint32_t*)t->inv,
           plan.pos, n, t->E, (const float*)t->hstage, t->deltas);
  std::vector<std::uint64_t> cnt(t->G, 0);
  std::vector<const std::uint64_t*> srckeys(t->G);
  std::vector<const float*> srcdel(t->G);
  if (t->G == 1) {
    cnt[0] = t->hsc->U;
    srckeys[0] = t->ukeys;
    srcdel[0] = t->deltas;
  } else {
    const int V = vec_of(t->E);
    const std::uint64_t work = t->Omax * std::uint64_t(t->E / V);
    if (V == 4)
      launch(t, p2p_send_deltas_kernel<4>, grid_for(work, 256, kSMs * 4), 256, 0, t->ctx, t->G,
             t->g, t->slot, (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
             (const std::uint32_t*)t->orank, (const float*)t->deltas, t->E, t->done_ctr);
    else
      launch(t, p2p_send_deltas_kernel<1>, grid_for(work, 256, kSMs * 4), 256, 0, t->ctx, t->G,
             t->g, t->slot, (const std::uint64_t*)t->ukeys, (const std::uint64_t*)&t->dsc->U,
             (const std::uint32_t*)t->orank, (const float*)t->deltas, t->E, t->done_ctr);
    p2p_wait(t, kPhDeltas);
    const int par = int(t->p2p_epoch & 1);
    std::vector<std::uint64_t> hdr(2 * t->G);
    HPS_CUDA(cudaMemcpyAsync(hdr.data(), t->w_hdr_p[par], hdr.size() * 8, cudaMemcpyDeviceToHost,
                             t->st));
    HPS_TRY(check_device_error(t, "device table: missing key ", true));
    for (int s = 0; s < t->G; ++s) {
      cnt[s] = hdr[2 * s];
      srckeys[s] = t->w_keys_p[par] + s * t->slot;
      srcdel[s] = t->w_deltas_p[par] + s * t->slot * t->E;
    }
  }
  if (dup) return set_error(HPS_ERR_ARG, "push: keys must be unique (a key->delta map)");
  const std::uint64_t E = std::uint64_t(t->E);
  std::uint64_t need = t->pend_used;
  for (int s = 0; s < t->G; ++s) need += cnt[s];
  if (need > t->pend_cap) {  // grow the arena (doubling), keeping what is pending
    const std::uint64_t nc = std::max<std::uint64_t>(need, 2 * t->pend_cap);
    std::uint64_t* nk = nullptr;
    float* nd = nullptr;
    HPS_CUDA(cudaMalloc(&nk, nc * 8));
    HPS_CUDA(cudaMalloc(&nd, nc * E * 4));
    if (t->pend_used) {
      HPS_CUDA(cudaMemcpyAsync(nk, t->pend_keys, t->pend_used * 8, cudaMemcpyDeviceToDevice, t->st));
      HPS_CUDA(cudaMemcpyAsync(nd, t->pend_deltas, t->pend_used * E * 4, cudaMemcpyDeviceToDevice,
                               t->st));
    }
    HPS_CUDA(cudaStreamSynchronize(t->st));
    cudaFree(t->pend_keys);
    cudaFree(t->pend_deltas);
    t->pend_keys = nk;
    t->pend_deltas = nd;
    t->pend_cap = nc;
  }
  for (int s = 0; s < t->G; ++s) {
    if (!cnt[s]) continue;
    PendingChunk c{s, cnt[s], t->pend_used};
    HPS_CUDA(cudaMemcpyAsync(t->pend_keys + c.at, srckeys[s], c.n * 8, cudaMemcpyDeviceToDevice,
                             t->st));
    HPS_CUDA(cudaMemcpyAsync(t->pend_deltas + c.at * E, srcdel[s], c.n * E * 4,
                             cudaMemcpyDeviceToDevice, t->st));
    t->pend_used += c.n;
    t->pending.push_back(c);
  }
  HPS_CUDA(cudaStreamSynchronize(t->st));
  return HPS_OK;
}

hps_status hps_drain(hps_tier_t t) {
  HPS_ENTER_Q(t);
  HPS_TRY(require_built(t));
  t->tab_flushed[t->cur] = false;  // its rows changed: written back again
  const int V = vec_of(t->E);
  for (int src : canonical_senders(t)) {
    for (auto& c : t->pending) {
      if (c.src != src) continue;
      const std::uint64_t work = c.n * std::uint64_t(t->E / V);
      if (V == 4)
        launch(t, table_apply_kernel<4>, grid_for(work), 256, 0,
               (const std::uint32_t*)nullptr, (const std::uint64_t*)(t->pend_keys + c.at),
               (const std::uint64_t*)t->tkeys[t->cur],
               (const std::uint64_t*)&t->dsc->cap[t->cur],
               (const float*)(t->pend_deltas + c.at * std::uint64_t(t->E)),
               (const std::uint64_t*)nullptr, c.n, t->tvals[t->cur], t->opt, &t->dsc->err);
      else
        launch(t, table_apply_kernel<1>, grid_for(work), 256, 0,
               (const std::uint32_t*)nullptr, (const std::uint64_t*)(t->pend_keys + c.at),
               (const std::uint64_t*)t->tkeys[t->cur],
               (const std::uint64_t*)&t->dsc->cap[t->cur],
               (const float*)(t->pend_deltas + c.at * std::uint64_t(t->E)),
               (const std::uint64_t*)nullptr, c.n, t->tvals[t->cur], t->opt, &t->dsc->err);
    }
  }
  const hps_status s = check_device_error(t, "device table: accumulate to missing key ");
  t->pending.clear();
  t->pend_used = 0;
  return s;
}

hps_status hps_apply_local(hps_tier_t t, const uint64_t* keys, const float* deltas, uint64_t n) {
  HPS_ENTER_Q(t);
  HPS_TRY(require_built(t));
  if (n > t->Omax)
    return set_error(HPS_ERR_CAPACITY, "apply: %llu keys exceed max_batch_keys",
                     (unsigned long long)n);
  if (!n) return HPS_OK;
  if (!keys || !deltas) return set_error(HPS_ERR_ARG, "null argument");
  t->tab_flushed[t->cur] = false;  // its rows change: written back again
  const std::uint64_t E = std::uint64_t(t->E);
  HPS_CUDA(cudaMemcpyAsync(t->lane[0].kB, keys, n * 8, cudaMemcpyHostToDevice, t->st));
  HPS_CUDA(cudaMemcpyAsync(t->hstage, deltas, n * E * 4, cudaMemcpyHostToDevice, t->st));
  const int V = vec_of(t->E);
  auto k = V == 4 ? table_apply_kernel<4> : table_apply_kernel<1>;
  launch(t, k, grid_for(n * std::uint64_t(t->E / V)), 256, 0, (const std::uint32_t*)nullptr,
         (const std::uint64_t*)t->lane[0].kB, (const std::uint64_t*)t->tkeys[t->cur],
         (const std::uint64_t*)&t->dsc->cap[t->cur], (const float*)t->hstage,
         (const std::uint64_t*)nullptr, n, t->tvals[t->cur], t->opt, &t->dsc->err);
  return check_device_error(t, "device table: accumulate to missing key ");
}

hps_status hps_table_info(hps_tier_t t, uint64_t* capacity, uint64_t* occupancy,
                          uint64_t* width) {
  HPS_ENTER_Q(t);
  HPS_TRY(require_built(t));
  HPS_CUDA(cudaMemcpyAsync(t->hsc->cap, t->dsc->cap, sizeof(t->dsc->cap), cudaMemcpyDeviceToHost,
                           t->st));
  HPS_CUDA(cudaMemcpyAsync(t->hsc->nws_tab, t->dsc->nws_tab, sizeof(t->dsc->nws_tab),
                           cudaMemcpyDeviceToHost, t->st));
  HPS_CUDA(cudaStreamSynchronize(t->st));
  if (capacity) *capacity = t->hsc->cap[t->cur];
  if (occupancy) *occupancy = t->hsc->nws_tab[t->cur];
  if (width) *width = std::uint64_t(t->E);
  return HPS_OK;
}

hps_status hps_row_width(hps_tier_t t, uint64_t* row_width) {
  if (!t || !row_width) return set_error(HPS_ERR_ARG, "null argument");
  *row_width = std::uint64_t(t->RW);
  return HPS_OK;
}

hps_status hps_table_lookup(hps_tier_t t, const uint64_t* keys, uint64_t n, uint8_t* found,
                            float* rows) {
  HPS_ENTER_Q(t);
  HPS_TRY(require_built(t));
  if (!n) return HPS_OK;
  if (!keys || !found) return set_error(HPS_ERR_ARG, "null argument");
  const std::uint64_t RW = std::uint64_t(t->RW);
  for (std::uint64_t c0 = 0; c0 < n; c0 += t->Omax) {  // chunks within the key scratch
    const std::uint64_t m = std::min(t->Omax, n - c0);
    HPS_TRY(ensure_staged(t, m * RW));
    auto* dfound = reinterpret_cast<std::uint8_t*>(t->lane[0].vB);  // (m bytes <= Omax x 4)
    HPS_CUDA(cudaMemcpyAsync(t->lane[0].kB, keys + c0, m * 8, cudaMemcpyHostToDevice, t->st));
    launch(t, table_lookup_kernel, grid_for(m), 256, 0, (const std::uint64_t*)t->lane[0].kB, m,
           (const std::uint64_t*)t->tkeys[t->cur], (const float*)t->tvals[t->cur],
           (const std::uint64_t*)&t->dsc->cap[t->cur], t->RW, dfound,
           rows ? t->staged : (float*)nullptr);
    HPS_CUDA(cudaMemcpyAsync(found + c0, dfound, m, cudaMemcpyDeviceToHost, t->st));
    if (rows)
      HPS_CUDA(cudaMemcpyAsync(rows + c0 * RW, t->staged, m * RW * 4, cudaMemcpyDeviceToHost,
                               t->st));
    HPS_CUDA(cudaStreamSynchronize(t->st));
  }
  return HPS_OK;
}

hps_status hps_table_slots(hps_tier_t t, uint64_t* slot_keys, float* rows) {
  std::uint64_t cap = 0;
  HPS_TRY(hps_table_info(t, &cap, nullptr, nullptr));
  if (slot_keys)
    HPS_CUDA(cudaMemcpyAsync(slot_keys, t->tkeys[t->cur], cap * 8, cudaMemcpyDeviceToHost, t->st));
  if (rows)
    HPS_CUDA(cudaMemcpyAsync(rows, t->tvals[t->cur], cap * std::uint64_t(t->RW) * 4,
                             cudaMemcpyDeviceToHost, t->st));
  HPS_CUDA(cudaStreamSynchronize(t->st));
  return HPS_OK;
}


hps_status hps_dump(hps_tier_t t, uint64_t* keys_out, float* rows_out, uint64_t* n_out) {
  std::uint64_t occ = 0, cap = 0;
  HPS_TRY(hps_table_info(t, &cap, &occ, nullptr));
  // the working set in key order: t->ws when the build sorted it, else sorted
  // here from the table itself into scratch (t->ws stays paired with ws_idx)
  const std::uint64_t* wsk = t->ws;
  if (!t->ws_sorted) {
    open_lookback_context(t);
    tile_scan(t, LiveSlot{t->tkeys[t->cur]},
              CompactEmit{t->tkeys[t->cur], nullptr, t->lane[0].kB, nullptr}, Count{nullptr, cap}, cap,
              &t->lane[0].d->total);
    std::uint64_t* sk = nullptr;
    std::uint32_t* so = nullptr;
    radix_sort(t, t->lane[0].kB, nullptr, Count{nullptr, occ}, occ, t->sort_bits, false, &sk, &so);
    wsk = sk;
  }
  const int V = vec_of(t->RW);
  const std::uint64_t work = occ * std::uint64_t(t->RW / V);
  if (occ) HPS_TRY(ensure_staged(t, occ * std::uint64_t(t->RW)));
  if (occ) {
    if (V == 4)
      launch(t, table_dump_kernel<4>, grid_for(work), 256, 0, wsk,
             (const std::uint64_t*)&t->dsc->nws_tab[t->cur], (const std::uint64_t*)t->tkeys[t->cur],
             (const float*)t->tvals[t->cur], (const std::uint64_t*)&t->dsc->cap[t->cur],
             (float*)nullptr, std::uint64_t(0), t->staged, t->RW, &t->dsc->err);
    else
      launch(t, table_dump_kernel<1>, grid_for(work), 256, 0, wsk,
             (const std::uint64_t*)&t->dsc->nws_tab[t->cur], (const std::uint64_t*)t->tkeys[t->cur],
             (const float*)t->tvals[t->cur], (const std::uint64_t*)&t->dsc->cap[t->cur],
             (float*)nullptr, std::uint64_t(0), t->staged, t->RW, &t->dsc->err);
    if (keys_out) HPS_CUDA(cudaMemcpyAsync(keys_out, wsk, occ * 8, cudaMemcpyDeviceToHost, t->st));
    if (rows_out)
      HPS_CUDA(cudaMemcpyAsync(rows_out, t->staged, occ * std::uint64_t(t->RW) * 4,
                               cudaMemcpyDeviceToHost, t->st));
  }
  HPS_TRY(check_device_error(t, "device table: missing key "));
  if (n_out) *n_out = occ;
  return HPS_OK;
}

hps_status hps_dense_sync(hps_tier_t t, float* buf, uint64_t len, int deterministic) {
  HPS_ENTER_Q(t);
  (void)deterministic;  // the canonical f64 sum serves both modes (hps_gpu.h)
  if (len == 0 || t->G == 1) return HPS_OK;  // a single replica is untouched
  const std::uint64_t nw = std::uint64_t(t->md.nw);
  float* sum = t->hstage;
  for (std::uint64_t c0 = 0; c0 < len; c0 += nw) {  // window-sized rounds
    const std::uint64_t L = std::min(nw, len - c0);
    HPS_CUDA(cudaMemsetAsync(t->dgrad, 0, nw * 4, t->st));
    HPS_CUDA(cudaMemcpyAsync(t->dgrad, buf + c0, L * 4, cudaMemcpyHostToDevice, t->st));
    begin_round(t);
    launch(t, p2p_send_dense_kernel, grid_for(nw * t->G), 256, 0, t->ctx, t->G, t->g, nw,
           (const float*)t->dgrad, t->done_ctr);
    launch(t, p2p_dense_update_kernel, 1, 256, 0, t->ctx, t->G, t->g, t->N, t->D, nw,
           (float*)nullptr, 1.0f, 0, sum, &t->dsc->err, int(kPhDense));
    HPS_CUDA(cudaMemcpyAsync(buf + c0, sum, L * 4, cudaMemcpyDeviceToHost, t->st));
  }
  return check_device_error(t, "device table: missing key ", true);
}

hps_status hps_dense_count(hps_tier_t t, uint64_t* n) {
  if (!t || !n) return set_error(HPS_ERR_ARG, "null argument");
  *n = std::uint64_t(t->md.nw);
  return HPS_OK;
}

hps_status hps_get_dense(hps_tier_t t, float* w) {
  HPS_ENTER_Q(t);
  HPS_CUDA(cudaMemcpyAsync(w, t->dense, std::uint64_t(t->md.nw) * 4, cudaMemcpyDeviceToHost, t->st));
  HPS_CUDA(cudaStreamSynchronize(t->st));
  return HPS_OK;
}

hps_status hps_set_dense(hps_tier_t t, const float* w) {
  HPS_ENTER_Q(t);
  HPS_CUDA(cudaMemcpyAsync(t->dense, w, std::uint64_t(t->md.nw) * 4, cudaMemcpyHostToDevice, t->st));
  HPS_CUDA(cudaStreamSynchronize(t->st));
  return HPS_OK;
}

hps_status hps_flush(hps_tier_t t) {
  HPS_ENTER_Q(t);  // (quiesce: in-flight batches done, every resident row queued)
  HPS_CUDA(cudaStreamSynchronize(t->st_wb));
  for (int p = 0; p < kTables; ++p) {
    wb_account(t, p, true);
    t->wb_pending[p] = false;
  }
  return HPS_OK;
}

hps_status hps_store_mode(hps_tier_t t, int* mode) {
  if (!t || !mode) return set_error(HPS_ERR_ARG, "null argument");
  *mode = !t->store ? HPS_STORE_NONE
          : t->mirror ? HPS_STORE_HOST_MIRRORED
          : !t->store_on_host ? HPS_STORE_DEVICE
          : t->dma ? HPS_STORE_HOST_DMA : HPS_STORE_HOST_ZEROCOPY;
  return HPS_OK;
}

hps_status hps_store_pcie_bytes(hps_tier_t t, uint64_t* h2d, uint64_t* d2h) {
  HPS_ENTER(t);
  std::uint64_t r = 0, w = 0;
  HPS_TRY(hps_store_traffic(t, &r, &w));
  const std::uint64_t rowb = std::uint64_t(t->RW) * 4;
  // zero-copy / DMA staging move every store row they read or write; the
  // mirror moves its attach copy and its copy-backs
  if (h2d) *h2d = t->mirror_h2d + (t->store_on_host ? r * rowb : 0);
  if (d2h) *d2h = t->mirror_d2h + (t->store_on_host ? w * rowb : 0);
  return HPS_OK;
}

hps_status hps_store_traffic(hps_tier_t t, uint64_t* rows_read, uint64_t* rows_written) {
  HPS_ENTER(t);
  HPS_CUDA(cudaMemcpyAsync(&t->hsc->wb_total, &t->dsc->wb_total, 8, cudaMemcpyDeviceToHost,
                           t->st_wb));
  HPS_CUDA(cudaStreamSynchronize(t->st_wb));
  if (rows_read) *rows_read = t->rows_read;
  if (rows_written) *rows_written = t->hsc->wb_total;
  return HPS_OK;
}

hps_status hps_attach_store(hps_tier_t t, float* rows, uint64_t num_keys, int on_device) {
  HPS_ENTER_Q(t);
  HPS_TRY(hps_flush(t));
  for (auto& kv : t->graphs) cudaGraphExecDestroy(kv.second.exec);
  t->graphs.clear();
  for (bool& f : t->tab_wb) f = false;  // earlier tables wrote to another store
  t->store_on_host = false;
  if (t->store_registered) {
    cudaHostUnregister(t->store_host);
    t->store_registered = false;
  }
  t->store = nullptr;
  t->store_keys = 0;
  t->store_hptr = nullptr;
  t->dma = false;
  if (t->mirror) {  // (hps_flush above copied it back)
    cudaFree(t->mirror);
    cudaFree(t->mirror_pages);
    if (t->mirror_registered) cudaHostUnregister(t->mirror_host);
    t->mirror_registered = false;
    t->mirror_hmapped = nullptr;
    t->mirror = nullptr;
    t->mirror_pages = nullptr;
    t->mirror_hpages.clear();
    t->mirror_host = nullptr;
    t->mirror_bytes = 0;
    t->mirror_dirty = false;
  }
  if (!rows || !num_keys) return HPS_OK;
  const std::uint64_t sbytes = num_keys * std::uint64_t(t->RW) * 4;
  std::size_t freeb = 0, totalb = 0;
  cudaMemGetInfo(&freeb, &totalb);
  // mirror when the store is small (the budget) or no bigger than 16 batches'
  // worst-case staging (then a run of ~16+ batches moves less over PCIe with
  // the one copy back than with per-batch staging; c3's 51 GB Adagrad store
  // vs its 3.3 GB working set), and it fits in HBM beside the tables
  const double wsb = double(t->Wmax) * double(t->RW) * 4.0;
  const bool worth = double(sbytes) <= t->mirror_gb * 1e9 || double(sbytes) <= 16.0 * wsb;
  // at G > 1 the ranks may share one host array: the copy-back then writes
  // only this rank's rows, through the array's device mapping (float4 rows)
  if ((t->G == 1 || t->RW % 4 == 0) && !on_device && t->stage_mode != 1 && t->mirror_gb > 0 &&
      worth && sbytes + (std::uint64_t(4) << 30) < freeb) {
    // the store fits in HBM: trained there, the host array exact when observed
    void* d = nullptr;
    void* pg = nullptr;
    const std::uint64_t np = ((num_keys - 1) >> kMirrorPageShift) + 1;
    if (t->G > 1) {
      cudaPointerAttributes at{};
      const bool pinned = cudaPointerGetAttributes(&at, rows) == cudaSuccess &&
                          at.type == cudaMemoryTypeHost;
      cudaGetLastError();
      if (!pinned) {
        HPS_CUDA(cudaHostRegister(rows, sbytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
        t->mirror_registered = true;
      }
      void* dp = nullptr;
      HPS_CUDA(cudaHostGetDevicePointer(&dp, rows, 0));
      t->mirror_hmapped = static_cast<float*>(dp);
    }
    if (cudaMalloc(&d, sbytes) == cudaSuccess && cudaMalloc(&pg, np) == cudaSuccess) {
      HPS_CUDA(cudaMemcpy(d, rows, sbytes, cudaMemcpyHostToDevice));
      HPS_CUDA(cudaMemset(pg, 0, np));
      t->mirror_h2d += sbytes;
      t->mirror_pages = static_cast<std::uint8_t*>(pg);
      t->mirror_hpages.assign(np, 0);
      t->mirror = static_cast<float*>(d);
      t->mirror_host = rows;
      t->mirror_bytes = sbytes;
      t->store = t->mirror;
      t->store_keys = num_keys;
      return HPS_OK;
    }
    if (d) cudaFree(d);
    if (t->mirror_registered) cudaHostUnregister(rows);
    t->mirror_registered = false;
    t->mirror_hmapped = nullptr;
    cudaGetLastError();
  }
  if (on_device) {
    t->store = rows;
  } else {
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, rows) == cudaSuccess &&
                        at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned) {
      HPS_CUDA(cudaHostRegister(rows, num_keys * std::uint64_t(t->RW) * 4,
                                cudaHostRegisterMapped | cudaHostRegisterPortable));
      t->store_registered = true;
      t->store_host = rows;
    }
    void* dp = nullptr;
    HPS_CUDA(cudaHostGetDevicePointer(&dp, rows, 0));
    t->store = static_cast<float*>(dp);
    t->store_on_host = true;
    t->store_hptr = rows;
    const std::uint64_t bytes = num_keys * std::uint64_t(t->RW) * 4;
    // measured (profiles/r2_bench_c5*.json, c3): bound-sized DMA + host-thread
    // copies lost to zero-copy on this box (c5 e2e 1.52M vs 1.60M ex/s, c3
    // 0.29M vs 0.55M), so zero-copy stays the default; HPS_STAGE=dma selects it
    (void)bytes;
    t->dma = t->stage_mode == 1;
    if (t->dma && !t->g_hrows) {  // pinned + device staging, once
      const std::uint64_t W = t->Wmax, RWb = std::uint64_t(t->RW) * 4;
      auto pin = [&](void** p, std::uint64_t b) {
        const cudaError_t e = cudaMallocHost(p, b);
        if (e == cudaSuccess) t->pinned.push_back(*p);
        return e;
      };
      void *a = nullptr, *b = nullptr, *c = nullptr, *d = nullptr, *e2 = nullptr, *f = nullptr;
      HPS_CUDA(pin(&a, 8));
      HPS_CUDA(pin(&b, W * 8));
      HPS_CUDA(pin(&c, W * RWb));
      HPS_CUDA(pin(&d, 8));
      HPS_CUDA(pin(&e2, W * 8));
      HPS_CUDA(pin(&f, W * RWb));
      t->g_hcnt = static_cast<std::uint64_t*>(a);
      t->g_hkeys = static_cast<std::uint64_t*>(b);
      t->g_hrows = static_cast<float*>(c);
      t->w_hcnt = static_cast<std::uint64_t*>(d);
      t->w_hkeys = static_cast<std::uint64_t*>(e2);
      t->w_hrows = static_cast<float*>(f);
      HPS_TRY(dalloc(t, &t->g_drows, W * std::uint64_t(t->RW)));
      HPS_TRY(dalloc(t, &t->w_drows, W * std::uint64_t(t->RW)));
    }
    const int threads =
        std::max(1, std::min(32, int(std::thread::hardware_concurrency()) / 2));
    t->gjob = Tier::DmaJob{t->g_hcnt, t->g_hkeys, t->g_hrows, rows, t->RW, threads, false};
    t->wjob = Tier::DmaJob{t->w_hcnt, t->w_hkeys, t->w_hrows, rows, t->RW, threads, true};
  }
  t->store_keys = num_keys;
  return HPS_OK;
}

hps_status hps_set_timing(hps_tier_t t, int enable) {
  HPS_ENTER_Q(t);
  t->timing = enable != 0;
  return HPS_OK;
}

hps_status hps_get_timing(hps_tier_t t, double* ms) {
  if (!t || !ms) return set_error(HPS_ERR_ARG, "null argument");
  for (int i = 0; i < HPS_TIMING_SLOTS; ++i) ms[i] = t->acc_ms[i];
  return HPS_OK;
}

hps_status hps_reset_timing(hps_tier_t t) {
  if (!t) return set_error(HPS_ERR_ARG, "null handle");
  for (double& v : t->acc_ms) v = 0;
  return HPS_OK;
}

hps_status hps_kernel_launches(hps_tier_t t, uint64_t* n) {
  if (!t || !n) return set_error(HPS_ERR_ARG, "null argument");
  *n = t->launches;
  return HPS_OK;
}

hps_status hps_debug_gemm_tf32(int M, int N, int K, const float* A, int64_t a_m, int64_t a_k,
                               const float* B, int64_t b_n, int64_t b_k, int b_ones_col, int epi,
                               float* D, double* Dd, int64_t ldd, const float* bias,
                               const float* mask, int64_t ldm, int splits) {
  if (M < 1 || N < 1 || K < 1 || !A || !B || (epi == kEpiF64 ? !Dd : !D))
    return set_error(HPS_ERR_ARG, "debug_gemm: bad arguments");
  static Tier scratch;  // launch bookkeeping only
  {
    const char* v = std::getenv("HPS_TF32_1X");
    scratch.gemm_split3 = !(v && std::atoi(v) != 0);
  }
  GemmArgs g{};
  g.M = M, g.N = N, g.K = K;
  g.A = A, g.a_m = a_m, g.a_k = a_k;
  g.B = B, g.b_n = b_n, g.b_k = b_k, g.b_ones_col = b_ones_col;
  g.epi = epi, g.D = D, g.Dd = Dd, g.ldd = ldd, g.bias = bias, g.mask = mask, g.ldm = ldm;
  for (int bn : {32, 64, 128}) {
    const int smem = int(gemm_smem(bn, true));
    if (bn == 32) cudaFuncSetAttribute(umma_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (bn == 64) cudaFuncSetAttribute(umma_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (bn == 128) cudaFuncSetAttribute(umma_gemm_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  launch_gemm(&scratch, nullptr, g, splits);
  HPS_CUDA(cudaGetLastError());
  HPS_CUDA(cudaDeviceSynchronize());
  return HPS_OK;
}

hps_status hps_graph_captures(hps_tier_t t, uint64_t* n) {
  if (!t || !n) return set_error(HPS_ERR_ARG, "null argument");
  *n = t->graph_captures;
  return HPS_OK;
}

hps_status hps_stream(hps_tier_t t, void** stream) {
  if (!t || !stream) return set_error(HPS_ERR_ARG, "null argument");
  *stream = t->st;
  return HPS_OK;
}

// ----------------------------------------------------- hps_train_batch

hps_status hps_submit_batch(hps_tier_t t, uint64_t B, const int64_t* offsets,
                            const uint64_t* keys, const uint8_t* labels, int on_device) {
  HPS_ENTER(t);
  if (!t->trace) return submit_batch(t, B, offsets, keys, labels, on_device, nullptr);
  const auto h0 = std::chrono::steady_clock::now();
  const hps_status s = submit_batch(t, B, offsets, keys, labels, on_device, nullptr);
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
  std::fprintf(stderr, "[trace] host submit %llu: %.0f us\n", (unsigned long long)(t->submitted - 1), us);
  return s;
}

hps_status hps_wait_batch(hps_tier_t t, hps_batch_stats* stats) {
  HPS_ENTER(t);
  if (t->done.empty()) {
    if (t->inflight.empty()) return set_error(HPS_ERR_ARG, "wait_batch: no batch in flight");
    const auto h0 = std::chrono::steady_clock::now();
    complete_oldest(t);
    if (t->trace)
      std::fprintf(stderr, "[trace] host wait: %.0f us\n",
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count());
  }
  Tier::Done d = std::move(t->done.front());
  t->done.pop_front();
  if (stats) *stats = d.stats;
  if (d.st != HPS_OK) return set_error(d.st, "%s", d.msg.c_str());
  return HPS_OK;
}

hps_status hps_train_batch(hps_tier_t t, uint64_t B, const int64_t* offsets,
                           const uint64_t* keys, const uint8_t* labels, int on_device,
                           hps_batch_stats* stats) {
  HPS_ENTER(t);
  std::uint64_t id = 0;
  HPS_TRY(submit_batch(t, B, offsets, keys, labels, on_device, &id));
  while (!t->inflight.empty() && t->inflight.front().id <= id) complete_oldest(t);
  for (auto it = t->done.begin(); it != t->done.end(); ++it) {
    if (it->id != id) continue;
    Tier::Done d = std::move(*it);
    t->done.erase(it);
    if (stats) *stats = d.stats;
    if (d.st != HPS_OK) return set_error(d.st, "%s", d.msg.c_str());
    return HPS_OK;
  }
  return set_error(HPS_ERR_ARG, "train_batch: lost batch %llu", (unsigned long long)id);
}

hps_status hps_set_graphs(hps_tier_t t, int enable) {
  if (!t) return set_error(HPS_ERR_ARG, "null handle");
  t->use_graphs = enable != 0;
  return HPS_OK;
}

}  // extern "C"
