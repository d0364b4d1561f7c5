// exchange.cpp -- halo exchange + rank-ordered reductions of the row-block
// partition: LocalGroup/LocalExchange (P ranks as threads of
// one process on one device, the one-GPU test vehicle) and NcclExchange (one rank
// per process, NCCL point-to-point + allgather; libnccl resolved at run time).
#include <dlfcn.h>

#include <cstring>

#include "engine.hpp"
#include "launch.hpp"

namespace f3rg {

static size_t esize(int p) { return p == 0 ? 2 : p == 1 ? 4 : 8; }

// ---- LocalGroup ----------------------------------------------------------------------
LocalGroup::LocalGroup(int p) : P(p) {
  if (P < 1) throw Error(ERR_DIMENSION, "local group: P must be >= 1");
  F3RG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  ptrs.assign((size_t)P, nullptr);
  all.alloc((size_t)P * 16 * sizeof(double));
  F3RG_CUDA(cudaMemset(all.get(), 0, all.bytes()));
}

LocalGroup::~LocalGroup() {
  if (stream) cudaStreamDestroy(stream);
}

void LocalGroup::set_plans(uint64_t n, const uint32_t* rp, const uint32_t* ci) {
  plans.clear();
  for (int r = 0; r < P; ++r) plans.push_back(make_plan(n, rp, ci, P, r));
  sidx.clear();
  sidx.resize((size_t)P);
  for (int q = 0; q < P; ++q) {
    sidx[q].resize((size_t)P);
    for (int p = 0; p < P; ++p) {
      const auto& v = plans[q].send_idx[p];
      if (v.empty()) continue;
      sidx[q][p].alloc(v.size() * 4);
      F3RG_CUDA(cudaMemcpy(sidx[q][p].get(), v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    }
  }
}

void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  if (failed_) throw Error(ERR_INTERNAL, "local group: a peer rank failed");
  const unsigned long long g = gen_;
  if (++arrived_ == P) {
    arrived_ = 0;
    ++gen_;
    cv_.notify_all();
    return;
  }
  cv_.wait(lk, [&] { return gen_ != g || failed_; });
  if (failed_) throw Error(ERR_INTERNAL, "local group: a peer rank failed");
}

void LocalGroup::fail() {
  std::lock_guard<std::mutex> lk(mu_);
  failed_ = true;
  cv_.notify_all();
}

// All ranks enqueue on the group's single stream, so stream order plus the two
// host barriers give the dependencies: every producer of the exchanged vector is
// enqueued before any gather reads it, and every gather before any rank's next
// write to its owned rows.
void LocalGroup::gather_into(int r, void* ext, int prec, cudaStream_t s) {
  const PartPlan& me = plans[r];
  const size_t es = esize(prec);
  for (int q = 0; q < P; ++q) {
    if (q == r || me.recv_cnt[q] == 0) continue;
    const char* src = static_cast<const char*>(ptrs[q]) + plans[q].off() * es;
    F3RG_CUDA(launch_gather(prec, Launch{0, s}, src, sidx[q][r].get<uint32_t>(), me.recv_cnt[q],
                            static_cast<char*>(ext) + me.recv_off[q] * es));
  }
}

void LocalExchange::halo(void* ext, int prec, cudaStream_t s) {
  g_->ptrs[r_] = ext;
  g_->barrier();
  g_->gather_into(r_, ext, prec, s);
  g_->barrier();
}

void LocalExchange::allgather(double*, double*, cudaStream_t) { g_->barrier(); }
void LocalExchange::done_reduce(cudaStream_t) { g_->barrier(); }

// ---- NCCL (runtime-resolved) ---------------------------------------------------------
namespace {
using ncclResult_t = int;
using ncclComm_t = void*;
struct ncclUniqueId {
  char internal[128];
};
enum { ncclUint8 = 1, ncclFloat64 = 8 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    const char* path = std::getenv("F3RG_NCCL_LIB");
    x.h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) throw Error(ERR_UNSUPPORTED, std::string("NCCL not loadable: ") + dlerror());
    auto sym = [&](const char* s) {
      void* p = dlsym(x.h, s);
      if (!p) throw Error(ERR_UNSUPPORTED, std::string("NCCL symbol missing: ") + s);
      return p;
    };
    x.GetUniqueId = reinterpret_cast<decltype(x.GetUniqueId)>(sym("ncclGetUniqueId"));
    x.CommInitRank = reinterpret_cast<decltype(x.CommInitRank)>(sym("ncclCommInitRank"));
    x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(sym("ncclCommDestroy"));
    x.Send = reinterpret_cast<decltype(x.Send)>(sym("ncclSend"));
    x.Recv = reinterpret_cast<decltype(x.Recv)>(sym("ncclRecv"));
    x.AllGather = reinterpret_cast<decltype(x.AllGather)>(sym("ncclAllGather"));
    x.GroupStart = reinterpret_cast<decltype(x.GroupStart)>(sym("ncclGroupStart"));
    x.GroupEnd = reinterpret_cast<decltype(x.GroupEnd)>(sym("ncclGroupEnd"));
    x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(sym("ncclGetErrorString"));
    return x;
  }();
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) throw Error(ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

void NcclExchange::unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

NcclExchange::NcclExchange(int P, int rank, const void* uid, uint64_t n, const uint32_t* rp, const uint32_t* ci)
    : plan_(make_plan(n, rp, ci, P, rank)) {
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  nccl_check(nccl().CommInitRank(&comm_, P, id, rank), "ncclCommInitRank");
  sidx_.resize((size_t)P);
  soff_.assign((size_t)P, 0);
  uint64_t tot = 0;
  for (int q = 0; q < P; ++q) {
    const auto& v = plan_.send_idx[q];
    soff_[q] = tot;
    tot += v.size();
    if (v.empty()) continue;
    sidx_[q].alloc(v.size() * 4);
    F3RG_CUDA(cudaMemcpy(sidx_[q].get(), v.data(), v.size() * 4, cudaMemcpyHostToDevice));
  }
  sendbuf_.alloc(tot * 8 + 16);
  loc_.alloc(16 * sizeof(double));
  all_.alloc((size_t)P * 16 * sizeof(double));
  F3RG_CUDA(cudaMemset(loc_.get(), 0, loc_.bytes()));
}

NcclExchange::~NcclExchange() {
  if (comm_) nccl().CommDestroy(comm_);
}

void NcclExchange::halo(void* ext, int prec, cudaStream_t s) {
  const size_t es = esize(prec);
  const int P = plan_.P;
  for (int q = 0; q < P; ++q)
    if (!plan_.send_idx[q].empty())
      F3RG_CUDA(launch_gather(prec, Launch{0, s}, static_cast<const char*>(ext) + plan_.off() * es,
                              sidx_[q].get<uint32_t>(), plan_.send_idx[q].size(),
                              sendbuf_.get<char>() + soff_[q] * es));
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int q = 0; q < P; ++q) {
    if (q == plan_.rank) continue;
    if (!plan_.send_idx[q].empty())
      nccl_check(nccl().Send(sendbuf_.get<char>() + soff_[q] * es, plan_.send_idx[q].size() * es, ncclUint8, q, comm_,
                             s),
                 "ncclSend");
    if (plan_.recv_cnt[q])
      nccl_check(nccl().Recv(static_cast<char*>(ext) + plan_.recv_off[q] * es, plan_.recv_cnt[q] * es, ncclUint8, q,
                             comm_, s),
                 "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

void NcclExchange::allgather(double* loc, double* all, cudaStream_t s) {
  nccl_check(nccl().AllGather(loc, all, 16, ncclFloat64, comm_, s), "ncclAllGather");
}

}  // namespace f3rg
