// f2v_internal.h -- the device context shared by the C-ABI and host driver
// (f2v_capi.cpp), the host data formats (f2v_graph.cpp) and the kernels
// (f2v_step.cu, f2v_epoch*.cu, f2v_perm.cu, f2v_walk.cu, f2v_shard.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <vector>

#include "../../include/force2vec_b200.h"

namespace f2v {

// Error raised inside the library; carries the C-ABI code.
struct Error {
  int32_t code;
  std::string msg;
};

[[noreturn]] void fail(int32_t code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define F2V_CUDA(x) ::f2v::cuda_check((x), #x)
// after a launch: launch errors always; with F2V_SYNC_DEBUG=1 also synchronise
// so an asynchronous fault is attributed to the kernel that caused it.
void launch_check(cudaStream_t s, const char* what);
#define F2V_LAUNCHED(stream, name) ::f2v::launch_check((stream), (name))

// Per-pair model parameters in the form the kernels use.
struct ForceParams {
  int32_t kind;
  int32_t has_cap;
  double eps;  // double(model.epsilon)   (force_kernels.cpp:105,113)
  double cap;  // double(*repulsion_cap)  (force_kernels.cpp:72)
  // epoch kernel: set to 1 when a Znew row never arrived within the poll
  // deadline (a stalled or dead peer GPU); the host raises F2V_ECUDA
  uint32_t* stall = nullptr;
};

struct DeviceBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t want);
  void release();
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Tunables of the dataflow epoch kernel; each can
// be overridden by the environment variable named beside it.
struct EpochTuning {
  uint32_t chunk = 256;  // F2V_CHUNK: max arcs per E item (hub splitting)
  uint32_t lgroup = 16;  // F2V_LGROUP: E chunks per L item
  uint32_t window = 48;  // F2V_WINDOW: arcs to batches [j-window, j) go to L items
  uint32_t recent = 8;   // F2V_RECENT: window arcs this recent are taken last
  uint32_t lwarps = 1;   // F2V_LWARPS: L-role warps per 8-warp CTA (autotuned 1 or 2 if unset)
  bool lwarps_env = false;
  uint32_t fast = 1;     // F2V_PRECISION=exact|fast: pair math precision (config)
  uint32_t ctas = 0;     // F2V_CTAS: resident epoch CTAs per SM (0 = as many as fit)
  uint32_t minb = 0;     // F2V_MINB: epoch register budget 2 or 3 CTAs/SM (0 = autotune)
};
void load_tuning(EpochTuning& t);

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  std::string err;
  uint64_t launches = 0;
  EpochTuning tune;

  // graph (CsrGraph, csr_graph.hpp:24-101)
  uint32_t n = 0;
  uint64_t nnz = 0;
  DeviceBuf rowptr, col;
  std::vector<uint64_t> h_rowptr;  // host copy: degrees for counters/partials
  // chunk / L-group layout, static per (graph, chunk, lgroup)
  DeviceBuf cbase, lbase, lpo, ecnt, lcnt, vflag;
  uint64_t chunks = 0, lgroups = 0, lslots = 0;
  uint32_t prepared_chunk = 0, prepared_lgroup = 0;

  // embedding (EmbeddingMatrix, trainer.hpp:33-57): double-buffered for epochs
  uint32_t d = 0;
  DeviceBuf z[2];
  int cur = 0;

  // per-step staging (GradBuffer, trainer.hpp:59-71)
  DeviceBuf grads, ids, negs, vloss, bad, scratch;
  uint32_t staged_b = 0;

  // epoch buffers
  DeviceBuf perm, state, negs_all, negwin, items, litems, nE, nL, EP, LP, wtot, needs, scan_tmp,
      epart, eloss, wcnt, wl, lpart, lloss, ploss, counters, pcnt, pslot;
  uint32_t last_litems = 0;
  // occupancy autotune (FAST d = 128): kernel ms of the 2- and 3-CTA builds on
  // this graph + config (negative = not yet timed) and the build in use
  double occ_ms[2] = {-1.0, -1.0};
  uint64_t occ_key = 0;
  uint32_t occ_epochs = 0;
  bool dry_launch = false;  // launch_epoch only loads the selected kernel
  int occ_use = 2;
  uint32_t occ_lwarps = 1;
  // vertex shards: G shards, step-major combined order
  uint32_t shards = 1;        // G of the current run
  int32_t rank = -1;          // this process's shard; -1 = one process runs every shard
  uint32_t world = 1;         // processes (GPUs) sharing the run through peer replicas
  DeviceBuf poff, lperm;      // combined start of (step, shard) batches; per-shard perms
  std::vector<uint32_t> h_poff;
  uint32_t steps = 0;         // T = max over shards of the local batch count
  // batch range of one epoch (f2v_train_config.first_batch / run_batches):
  // positions [range_p0, range_p1) = steps [range_t0, range_t1); others keep Z
  uint32_t range_p0 = 0, range_p1 = 0, range_t0 = 0, range_t1 = 0;
  bool ranged = false;
  uint64_t layout_key[4] = {0, 0, 0, 0};  // (graph_gen, batch, G, s) of the layout
  uint64_t graph_gen = 0;                  // bumped by every f2v_upload_graph
  std::vector<uint32_t> sh_lo, sh_bs, sh_nb;  // per shard: first row, batch, batches
  // multi-process: IPC-shared control block + the peers' replicas (f2v_shard.cu)
  DeviceBuf ctl;
  // per-step all-gather baseline (f2v_nccl.cu): NCCL communicator + packs
  void* nccl_comm = nullptr;
  uint32_t nccl_rank = 0, nccl_world = 1;
  DeviceBuf ag_send, ag_recv, ag_state;
  DeviceBuf rep[7];  // emulated peer replicas of Znew (F2V_EMULATE_REPLICAS, tests)
  bool shard_ready = false;
  float* peer_z[8][2] = {};
  void* peer_ctl[8] = {};
  void* peer_base[8][3] = {};  // IPC mappings to close
  uint64_t barriers = 0;
  // walk mode (f2v_walk.cu): while walk_k > 0, rowptr/col/h_rowptr/nnz hold
  // the per-epoch walk context and the graph CSR is parked here
  uint32_t walk_k = 0;
  DeviceBuf grow, gcol, wflag, wpos;
  std::vector<uint64_t> h_growptr;
  uint64_t gnnz = 0;
  DeviceBuf trace;  // DEBUG: per-position finalise timestamps (F2V_TRACE)
  DeviceBuf shufR, shufL;  // device Fisher-Yates (f2v_perm.cu)

  // back-to-back epochs (k_async_begin): the device run record and one
  // event pair per epoch kernel
  DeviceBuf runst;
  std::vector<cudaEvent_t> ev_async;
  // timing of the last train_epochs call (f2v_last_timing)
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  std::vector<cudaEvent_t> ev_kernel;  // pairs around each epoch kernel
  uint32_t ev_used = 0;
  double timing[4] = {0, 0, 0, 0};

  float* zcur() const { return z[cur].as<float>(); }
};

// kernels
void k_grad_minibatch(Ctx& c, uint32_t b, uint32_t s, const ForceParams& fp, bool want_loss);
void k_apply_update(Ctx& c, uint32_t b, float eta, bool unique_ids);
double k_batch_loss_sum(Ctx& c, uint32_t b);
void k_uniform_embedding(Ctx& c, uint64_t seed, float lo, float hi, int keyed_init);
// one device-resident epoch; returns the first failing perm position or UINT64_MAX
struct EpochResult {
  uint64_t bad_pos;
  double loss;
};
// Epochs of one f2v_train_epochs call run back to back with no host sync
// (k_epoch_run with slot >= 0): each epoch's outcome lands in a device run
// record; the first failure stops every later kernel and restores Z on the
// device; the host reads the record once at the end (k_async_finish).
struct AsyncOutcome {
  bool failed = false, stalled = false;
  uint32_t slot = 0, vertex = 0;
  uint64_t step = 0, pos = 0;
};
void k_async_begin(Ctx& c, uint32_t nslots);
AsyncOutcome k_async_finish(Ctx& c, uint32_t nslots, double* loss_out);
void k_prepare_graph(Ctx& c);
void k_shard_layout(Ctx& c, uint32_t batch, uint32_t G, uint32_t s);
void k_epoch_perm(Ctx& c, uint32_t epoch, uint64_t seed);
void k_epoch_begin(Ctx& c, uint32_t s, uint32_t epoch, uint64_t seed, int sampler);
void k_set_context(Ctx& c, uint32_t walk_k);   // f2v_walk.cu
void k_epoch_walks(Ctx& c, uint32_t epoch, uint64_t seed);
EpochResult k_epoch_run(Ctx& c, uint32_t s, float eta, const ForceParams& fp, bool monitor,
                        int async_slot = -1);
void k_epoch_restore(Ctx& c, uint64_t bad_step);
void k_device_partition(Ctx& c, uint32_t n, uint64_t seed, uint32_t epoch, uint32_t* perm_out);
void k_device_partition_keyed(Ctx& c, uint32_t n, uint64_t s0, uint32_t* perm_out);
// host: per-shard ranges/batches and the combined (step, shard) start positions
void shard_layout(const uint64_t* rowptr, uint32_t n, uint32_t s, uint32_t batch, uint32_t G,
                  std::vector<uint32_t>& lo,
                  std::vector<uint32_t>& bs, std::vector<uint32_t>& nb,
                  std::vector<uint32_t>& poff, uint32_t& T);
// multi-process shards (f2v_shard.cu)
void k_shard_barrier(Ctx& c);
void k_shard_publish(Ctx& c, uint64_t bad, double loss);
void k_shard_collect(Ctx& c, uint64_t& bad, double& loss);
size_t shard_ctl_bytes();
void k_rows(Ctx& c, uint32_t b, float* rows_dev, bool to_z);  // rows <-> Z[c.ids]

ForceParams make_params(const f2v_force_model& m);

// CsrGraph::from_edges on the device (f2v_csr.cu)
void device_csr_from_edges(cudaStream_t st, int num_sms, const uint32_t* pairs_host, uint64_t m,
                           uint32_t n, bool symmetrize, DeviceBuf& rowptr_dev, DeviceBuf& col_dev,
                           uint64_t* nnz_out, uint64_t* dups_out, uint64_t* loops_out);

// per-step all-gather baseline (f2v_nccl.cu)
struct AgResult {
  bool failed;
  uint32_t step, rank, index, vertex;
  double loss;
};
void nccl_unique_id(uint8_t* out128);
void k_nccl_init(Ctx& c, const uint8_t* id128, uint32_t rank, uint32_t world);
void k_nccl_destroy(Ctx& c);
void k_epoch_negatives(Ctx& c, uint32_t s, uint32_t epoch, uint64_t seed, int sampler);
AgResult k_allgather_epoch(Ctx& c, uint32_t s, float eta, const ForceParams& fp, bool monitor,
                           bool fast);


// the C-ABI wrapper pattern: run fn, map f2v::Error to its code and message
int32_t guard(Ctx* c, const std::function<void()>& fn);

// evaluation after training (f2v_eval.cu; evaluation.cpp in the reference)
namespace ev {
double kmeans(Ctx& c, const float* z, uint64_t n, uint32_t d, int k, uint64_t& rng, int restarts,
              int max_iters, int32_t* assign_host);
double kmeans_inertia(Ctx& c, const float* z, uint64_t n, uint32_t d, int k,
                      const int32_t* assign_host);
double modularity(Ctx& c, int k, const int32_t* assign_host);
void fit_logreg(Ctx& c, const float* x_host, uint64_t n, uint32_t d, const int32_t* targets,
                double lr, int iters, double l2, double* weights_out);
double logreg_loss(Ctx& c, const double* weights, const float* x_host, uint64_t n, uint32_t d,
                   const int32_t* targets, double l2);
double link_accuracy(Ctx& c, const float* z, uint32_t d, const uint32_t* train_pairs,
                     uint64_t ntrain, const uint32_t* test_pairs, uint64_t ntest, double lr,
                     int iters, double l2, double* weights_out);
void one_vs_rest(Ctx& c, const float* z, uint32_t d, const uint32_t* train_ids, uint64_t ntrain,
                 const uint32_t* test_ids, uint64_t ntest, uint32_t M, const uint8_t* tgt,
                 double lr, int iters, double l2, double* weights_out, double* prob_out);
}  // namespace ev

}  // namespace f2v

struct f2v_ctx {
  f2v::Ctx c;
};
