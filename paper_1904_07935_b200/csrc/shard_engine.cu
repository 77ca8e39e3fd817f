// The sharded engine: one engine per GPU, rank g of `world`
// owns the W rows [v_lo, v_hi) and the Ht rows [d_lo, d_hi) of balanced
// contiguous splits, A's CSR row block A[v_lo:v_hi, :] and the CSR of A^T's
// row block A^T[d_lo:d_hi, :] (transpose() order, proj/src/csr_matrix.cpp:30-50).
//
// Per iteration (the reference's order, proj/src/solver.cpp:79-92), with the
// hooks in engine.cu:
//   precompute_h   wait for every rank's W rows (pushed at the end of the last W
//                  update) -> R_g = A^T[d_lo:d_hi, :] W_full; S = sum_g gram(W_g)
//                  in rank order (push the K x K partial into every window, wait,
//                  add the world's partials in rank order)
//   update_h       row-local (hals.cpp / tiled.cpp on the local rows), then push
//                  the new Ht rows into every window
//   precompute_w   wait for Ht; P_g = A[v_lo:v_hi, :] Ht_full; Q = sum_g gram(Ht_g)
//   update_w       the streaming tiled kernel on the local rows; each column's
//                  norm = sqrt(sum_g ||W_g[:, t]||^2) exchanged INSIDE the
//                  persistent kernel over peer memory (peer.cuh: world_sum —
//                  tiled.cpp:129-146 across GPUs); then push the new W rows
//   error          <P, W> summed over ranks in rank order, <S, Q> redundant
// There is no host synchronisation inside an iteration and no NCCL on the
// data path: every exchange is a store into the peer's window (NVLink P2P
// through CUDA IPC) ordered by release/acquire epoch flags.  The result is
// deterministic for a fixed world size and bit-identical on every rank.
//
// The full factors live in the window padded to world * cap rows (rank g's
// rows at g * cap), so a rank's slice is a fixed offset in every window; the
// shard blocks' column indices are remapped onto those positions once, at
// creation.
#include <cstring>

#include "engine.hpp"

namespace plnmf {
namespace shard {
namespace {

size_t wbytes(const plnmf_gpu_engine* e) { return sizeof(double) * (size_t)(e->world * e->vcap * e->k); }
size_t hbytes(const plnmf_gpu_engine* e) { return sizeof(double) * (size_t)(e->world * e->dcap * e->k); }

char* section(plnmf_gpu_engine* e, int p, size_t off) { return e->peer_win[p] + off; }

int* error_word(plnmf_gpu_engine* e) { return reinterpret_cast<int*>(e->win + e->lay.off_error); }

PeerPtrs flag_slots(plnmf_gpu_engine* e, PeerChannel c) {
    PeerPtrs f{};
    for (int p = 0; p < e->world; ++p)
        f.p[p] = section(e, p, e->lay.off_agflags + sizeof(unsigned) * (size_t)(c * kMaxWorld + e->rank));
    return f;
}

void require_connected(const plnmf_gpu_engine* e) {
    if (e->world > 1 && !e->connected)
        throw std::invalid_argument("sharded engine: ranks not connected (plnmf_gpu_shard_connect)");
}

// push `bytes` from src into section offset `off` (+ this rank's slot) of every window
void push(plnmf_gpu_engine* e, PeerChannel c, const void* src, size_t bytes, size_t off, bool skip_self) {
    require_connected(e);
    PeerPtrs dst{};
    for (int p = 0; p < e->world; ++p) dst.p[p] = section(e, p, off);
    const unsigned epoch = ++e->ag_epoch[c];
    e->launches += kern::peer_push(e->s, src, (int64_t)bytes, dst, e->world, e->rank, skip_self, flag_slots(e, c),
                                   epoch, e->push_done, e->sms);
}

}  // namespace

double* w_full(const plnmf_gpu_engine* e) {
    char* b0 = e->win + e->lay.off_wfull[0];
    const char* w = reinterpret_cast<const char*>(e->w);
    return reinterpret_cast<double*>((w >= b0 && w < b0 + wbytes(e)) ? b0 : e->win + e->lay.off_wfull[1]);
}

double* ht_full(const plnmf_gpu_engine* e) {
    char* b0 = e->win + e->lay.off_hfull[0];
    const char* h = reinterpret_cast<const char*>(e->ht);
    return reinterpret_cast<double*>((h >= b0 && h < b0 + hbytes(e)) ? b0 : e->win + e->lay.off_hfull[1]);
}

void wait(plnmf_gpu_engine* e, PeerChannel c) {
    if (e->world == 1) return;
    require_connected(e);
    const unsigned* flags = reinterpret_cast<const unsigned*>(e->win + e->lay.off_agflags) + c * kMaxWorld;
    e->launches += kern::peer_wait(e->s, flags, e->world, e->ag_epoch[c], error_word(e), e->peer_timeout_ns);
}

void push_factor(plnmf_gpu_engine* e, PeerChannel c) {
    if (e->world == 1) return;
    if (c == kChanW) {
        const size_t off = (size_t)(reinterpret_cast<char*>(e->w) - e->win);  // this rank's slice of the full W
        push(e, c, e->w, sizeof(double) * (size_t)(e->v * e->k), off, true);
    } else {
        const size_t off = (size_t)(reinterpret_cast<char*>(e->ht) - e->win);
        push(e, c, e->ht, sizeof(double) * (size_t)(e->d * e->k), off, true);
    }
}

void reduce_kxk(plnmf_gpu_engine* e, PeerChannel c, double* inout) {
    if (e->world == 1) return;
    const int64_t kk = e->k * e->k;
    const size_t base = c == kChanS ? e->lay.off_sparts : e->lay.off_qparts;
    push(e, c, inout, sizeof(double) * (size_t)kk, base + sizeof(double) * (size_t)(e->rank * kk), false);
    wait(e, c);
    e->launches += kern::sum_parts(e->s, reinterpret_cast<const double*>(e->win + base), e->world, kk, kk, inout);
}

void reduce_scalar(plnmf_gpu_engine* e, double* inout) {
    if (e->world == 1) return;
    push(e, kChanPW, inout, sizeof(double), e->lay.off_pw + sizeof(double) * (size_t)e->rank, false);
    wait(e, kChanPW);
    e->launches += kern::sum_parts(e->s, reinterpret_cast<const double*>(e->win + e->lay.off_pw), e->world, 1, 1, inout);
}

FusedPush fused_push(plnmf_gpu_engine* e, PeerChannel c, const double* out_local) {
    require_connected(e);
    FusedPush f;
    f.world = e->world;
    f.rank = e->rank;
    f.epoch = ++e->ag_epoch[c];
    f.done = e->push_done;
    const size_t off = (size_t)(reinterpret_cast<const char*>(out_local) - e->win);
    const PeerPtrs flags = flag_slots(e, c);
    for (int p = 0; p < e->world; ++p) {
        f.dst[p] = reinterpret_cast<double*>(section(e, p, off));
        f.flag[p] = static_cast<unsigned*>(flags.p[p]);
    }
    return f;
}

WorldXch next_exchange(plnmf_gpu_engine* e) {
    WorldXch x;
    x.world = e->world;
    x.rank = e->rank;
    if (e->world == 1) return x;
    require_connected(e);
    x.epoch = ++e->xch_epoch;
    x.timeout_ns = e->peer_timeout_ns;
    x.error = error_word(e);
    for (int p = 0; p < e->world; ++p) {
        x.vals[p] = reinterpret_cast<double*>(section(e, p, e->lay.off_xvals));
        x.flags[p] = reinterpret_cast<unsigned*>(section(e, p, e->lay.off_xflags));
    }
    return x;
}

void check_error(plnmf_gpu_engine* e) {
    if (e->world == 1) return;
    int err = 0;
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(&err, error_word(e), sizeof(int), cudaMemcpyDeviceToHost, e->s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    if (err)
        throw DeviceError("sharded engine: a peer rank did not arrive within the exchange timeout "
                          "(ranks out of step or a rank failed)");
}

void close_peers(plnmf_gpu_engine* e) {
    for (int p = 0; p < kMaxWorld; ++p)
        if (e->peer_ipc[p] && e->peer_win[p]) cudaIpcCloseMemHandle(e->peer_win[p]);
}

}  // namespace shard

namespace {

using plnmf::dalloc;
using plnmf::guarded;

std::pair<int64_t, int64_t> split(int64_t n, int world, int g) {
    const int64_t base = n / world, extra = n % world;
    const int64_t lo = g * base + std::min<int64_t>(g, extra);
    return {lo, lo + base + (g < extra ? 1 : 0)};
}

// ranges, window, workspace; the caller provides the blocks
void shard_init(plnmf_gpu_engine* e, int world, int rank, int64_t v, int64_t d) {
    if (world < 1 || world > kMaxWorld)
        throw std::invalid_argument("plnmf_gpu_create_shard: world must be in [1, 8]");
    if (rank < 0 || rank >= world) throw std::invalid_argument("plnmf_gpu_create_shard: shard rank out of range");
    if (v < 0 || d < 0) throw std::invalid_argument("CsrMatrix: negative dimension");
    if (v > INT32_MAX || d > INT32_MAX) throw std::invalid_argument("plnmf_gpu_create_shard: dimensions exceed int32");
    e->shard = true;
    e->world = world;
    e->rank = rank;
    e->vfull = v;
    e->dfull = d;
    const auto vr = split(v, world, rank), dr = split(d, world, rank);
    e->v_lo = vr.first;
    e->d_lo = dr.first;
    e->v = vr.second - vr.first;
    e->d = dr.second - dr.first;
    e->vcap = (v + world - 1) / world;
    e->dcap = (d + world - 1) / world;
    if (world * e->vcap > INT32_MAX || world * e->dcap > INT32_MAX)
        throw std::invalid_argument("plnmf_gpu_create_shard: dimensions exceed int32");
    e->sparse = true;
    e->lay = kern::peer_layout(world, e->vcap, e->dcap, e->k);
    e->win = dalloc<char>(e, (int64_t)e->lay.total);  // cudaMalloc: IPC-exportable
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->win, 0, e->lay.total, e->s));  // padded rows, flags and epochs at 0
    e->peer_win[rank] = e->win;
    e->push_done = dalloc<unsigned>(e, 1);
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->push_done, 0, sizeof(unsigned), e->s));
    const size_t wslice = sizeof(double) * (size_t)(rank * e->vcap * e->k);
    const size_t hslice = sizeof(double) * (size_t)(rank * e->dcap * e->k);
    e->w = reinterpret_cast<double*>(e->win + e->lay.off_wfull[0] + wslice);
    e->w_new = reinterpret_cast<double*>(e->win + e->lay.off_wfull[1] + wslice);
    e->ht = reinterpret_cast<double*>(e->win + e->lay.off_hfull[0] + hslice);
    e->h_new = reinterpret_cast<double*>(e->win + e->lay.off_hfull[1] + hslice);
    e->a2 = std::numeric_limits<double>::quiet_NaN();  // set by the caller (plnmf_gpu_shard_set_norm_sq)
}

void upload_block(plnmf_gpu_engine* e, int64_t rows, int64_t nnz, const int64_t* rp, const int64_t* ci,
                  const double* val, int64_t*& drp, int32_t*& dci, double*& dval) {
    std::vector<int32_t> ci32(nnz > 0 ? nnz : 1);
    for (int64_t i = 0; i < nnz; ++i) ci32[i] = (int32_t)ci[i];
    drp = dalloc<int64_t>(e, rows + 1);
    dci = dalloc<int32_t>(e, nnz);
    dval = dalloc<double>(e, nnz);
    PLNMF_CUDA_CHECK(cudaMemcpy(drp, rp, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice));
    if (nnz > 0) {
        PLNMF_CUDA_CHECK(cudaMemcpy(dci, ci32.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
        PLNMF_CUDA_CHECK(cudaMemcpy(dval, val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
}

// global indices -> padded window positions; then the workspace
void shard_finish(plnmf_gpu_engine* e) {
    e->launches += kern::remap_split_index(e->s, e->ci, e->nnz, e->dfull, e->world, e->dcap);
    e->launches += kern::remap_split_index(e->s, e->tci, e->nnz_t, e->vfull, e->world, e->vcap);
    eng::alloc_workspace(e);
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
}

template <class T>
void adopt(plnmf_gpu_engine* e, T* ptr, int64_t n) {
    e->allocs.push_back(ptr);
    e->bytes += (int64_t)(sizeof(T) * (size_t)std::max<int64_t>(1, n));
}

void validate_block(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci, const double* val) {
    // CsrMatrix::validate, proj/src/csr_matrix.cpp:8-28 (same messages)
    if (!rp) throw std::invalid_argument("CsrMatrix: row_ptr length must be rows+1");
    if (rp[0] != 0 || rp[rows] != nnz) throw std::invalid_argument("CsrMatrix: row_ptr must start at 0 and end at nnz");
    if (nnz > 0 && (!ci || !val)) throw std::invalid_argument("CsrMatrix: col_idx and values lengths differ");
    for (int64_t r = 0; r < rows; ++r) {
        if (rp[r] > rp[r + 1]) throw std::invalid_argument("CsrMatrix: row_ptr must be non-decreasing");
        for (int64_t i = rp[r]; i < rp[r + 1]; ++i) {
            if (ci[i] < 0 || ci[i] >= cols) throw std::invalid_argument("CsrMatrix: column index out of range");
            if (i > rp[r] && ci[i] <= ci[i - 1])
                throw std::invalid_argument("CsrMatrix: column indices must be strictly increasing per row");
            if (!std::isfinite(val[i]) || val[i] < 0.0)
                throw std::invalid_argument("CsrMatrix: values must be finite and non-negative");
        }
    }
}

// Ranks sharing one device wait on one another's kernels; under CUDA's lazy
// module loading, the first launch of a kernel may wait for the context to go
// idle — i.e. for another rank's spinning kernel — and never return.  Such
// processes must load eagerly (CUDA_MODULE_LOADING=EAGER).
bool lazy_module_loading() {
    using GetMode = int (*)(int*);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        cudaGetLastError();
        return true;  // unknown: assume the CUDA 12 default
    }
    int mode = 0;
    if (reinterpret_cast<GetMode>(fn)(&mode) != 0) return true;
    return mode != 1;  // CU_MODULE_EAGER_LOADING
}

}  // namespace
}  // namespace plnmf

using plnmf::guarded;

extern "C" {

plnmf_status plnmf_gpu_create_shard(int32_t device, int32_t world, int32_t shard_rank, int64_t v, int64_t d,
                                    int64_t nnz_rows, const int64_t* rp_rows, const int64_t* ci_rows,
                                    const double* val_rows, int64_t nnz_cols, const int64_t* rp_cols,
                                    const int64_t* ci_cols, const double* val_cols, double a_norm_sq, int64_t rank,
                                    plnmf_gpu_engine** out) {
    plnmf_gpu_engine* e = nullptr;
    const plnmf_status st = guarded([&] {
        if (!out) throw std::invalid_argument("plnmf_gpu_create_shard: null output");
        e = new plnmf_gpu_engine();
        plnmf::eng::setup_common(e, device, rank);
        plnmf::shard_init(e, world, shard_rank, v, d);
        plnmf::validate_block(e->v, d, nnz_rows, rp_rows, ci_rows, val_rows);
        plnmf::validate_block(e->d, v, nnz_cols, rp_cols, ci_cols, val_cols);
        e->nnz = nnz_rows;
        e->nnz_t = nnz_cols;
        e->a2 = a_norm_sq;
        plnmf::upload_block(e, e->v, nnz_rows, rp_rows, ci_rows, val_rows, e->rp, e->ci, e->val);
        plnmf::upload_block(e, e->d, nnz_cols, rp_cols, ci_cols, val_cols, e->trp, e->tci, e->tval);
        plnmf::shard_finish(e);
        *out = e;
    });
    if (st != PLNMF_OK) plnmf::eng::release(e);
    return st;
}

plnmf_status plnmf_gpu_create_shard_synthetic(int32_t device, int32_t world, int32_t shard_rank, int64_t v, int64_t d,
                                              double density, uint64_t seed, int64_t rank, plnmf_gpu_engine** out) {
    plnmf_gpu_engine* e = nullptr;
    const plnmf_status st = guarded([&] {
        if (!out) throw std::invalid_argument("plnmf_gpu_create_shard_synthetic: null output");
        e = new plnmf_gpu_engine();
        plnmf::eng::setup_common(e, device, rank);
        plnmf::shard_init(e, world, shard_rank, v, d);
        int64_t* rp = nullptr;
        int32_t* ci = nullptr;
        double* val = nullptr;
        e->nnz = plnmf::kern::synth_csr_device(e->s, e->v, d, density, seed, &rp, &ci, &val, e->v_lo);
        plnmf::adopt(e, rp, e->v + 1);
        plnmf::adopt(e, ci, e->nnz);
        plnmf::adopt(e, val, e->nnz);
        e->rp = rp;
        e->ci = ci;
        e->val = val;
        e->nnz_t = plnmf::kern::synth_transpose_block_device(e->s, v, d, density, seed, e->d_lo, e->d_lo + e->d, &rp,
                                                             &ci, &val);
        plnmf::adopt(e, rp, e->d + 1);
        plnmf::adopt(e, ci, e->nnz_t);
        plnmf::adopt(e, val, e->nnz_t);
        e->trp = rp;
        e->tci = ci;
        e->tval = val;
        e->launches += 6;
        plnmf::shard_finish(e);
        *out = e;
    });
    if (st != PLNMF_OK) plnmf::eng::release(e);
    return st;
}

plnmf_status plnmf_gpu_shard_info(const plnmf_gpu_engine* e, int32_t* world, int32_t* shard_rank, int64_t* v_lo,
                                  int64_t* v_hi, int64_t* d_lo, int64_t* d_hi) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("plnmf_gpu: null engine");
        if (!e->shard) throw std::invalid_argument("plnmf_gpu_shard_info: not a sharded engine");
        if (world) *world = e->world;
        if (shard_rank) *shard_rank = e->rank;
        if (v_lo) *v_lo = e->v_lo;
        if (v_hi) *v_hi = e->v_lo + e->v;
        if (d_lo) *d_lo = e->d_lo;
        if (d_hi) *d_hi = e->d_lo + e->d;
    });
}

plnmf_status plnmf_gpu_shard_norm_sq(plnmf_gpu_engine* e, double start, double* out) {
    return guarded([&] {
        plnmf::eng::check_engine(e);
        if (!e->shard || !out) throw std::invalid_argument("plnmf_gpu_shard_norm_sq: not a sharded engine");
        // InputMatrix's serial sum (proj/src/input_matrix.cpp:15-20) continued over this rank's rows
        constexpr int64_t kChunk = 1 << 23;
        std::vector<double> host((size_t)std::min<int64_t>(kChunk, std::max<int64_t>(1, e->nnz)));
        double n2 = start;
        for (int64_t b = 0; b < e->nnz; b += kChunk) {
            const int64_t m = std::min(kChunk, e->nnz - b);
            PLNMF_CUDA_CHECK(cudaMemcpy(host.data(), e->val + b, sizeof(double) * m, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < m; ++i) n2 += host[i] * host[i];
        }
        *out = n2;
    });
}

plnmf_status plnmf_gpu_shard_set_norm_sq(plnmf_gpu_engine* e, double a_norm_sq) {
    return guarded([&] {
        plnmf::eng::check_engine(e);
        if (!e->shard) throw std::invalid_argument("plnmf_gpu_shard_set_norm_sq: not a sharded engine");
        e->a2 = a_norm_sq;
    });
}

plnmf_status plnmf_gpu_shard_ipc_handle(plnmf_gpu_engine* e, void* handle) {
    return guarded([&] {
        plnmf::eng::check_engine(e);
        if (!e->shard || !handle) throw std::invalid_argument("plnmf_gpu_shard_ipc_handle: not a sharded engine");
        cudaIpcMemHandle_t h;
        PLNMF_CUDA_CHECK(cudaIpcGetMemHandle(&h, e->win));
        static_assert(sizeof(h) == PLNMF_IPC_HANDLE_BYTES, "CUDA IPC handle size");
        std::memcpy(handle, &h, sizeof(h));
    });
}

plnmf_status plnmf_gpu_shard_connect(plnmf_gpu_engine* e, const void* handles) {
    return guarded([&] {
        plnmf::eng::check_engine(e);
        if (!e->shard || !handles) throw std::invalid_argument("plnmf_gpu_shard_connect: not a sharded engine");
        if (e->connected) throw std::invalid_argument("plnmf_gpu_shard_connect: already connected");
        for (int p = 0; p < e->world; ++p) {
            if (p == e->rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char*>(handles) + (size_t)p * sizeof(h), sizeof(h));
            void* ptr = nullptr;
            PLNMF_CUDA_CHECK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            e->peer_win[p] = static_cast<char*>(ptr);
            e->peer_ipc[p] = true;
        }
        e->connected = true;
    });
}

plnmf_status plnmf_gpu_shard_set_timeout(plnmf_gpu_engine* e, double seconds) {
    return guarded([&] {
        plnmf::eng::check_engine(e);
        if (!e->shard || !(seconds > 0.0)) throw std::invalid_argument("plnmf_gpu_shard_set_timeout: bad argument");
        e->peer_timeout_ns = (unsigned long long)(seconds * 1e9);
    });
}

plnmf_status plnmf_gpu_shard_connect_local(plnmf_gpu_engine* const* engines, int32_t world) {
    return guarded([&] {
        if (!engines || world < 1 || world > plnmf::kMaxWorld)
            throw std::invalid_argument("plnmf_gpu_shard_connect_local: bad argument");
        bool one_device = true;
        for (int g = 0; g < world; ++g) {
            const plnmf_gpu_engine* e = engines[g];
            if (!e || !e->shard || e->world != world || e->rank != g || e->connected)
                throw std::invalid_argument("plnmf_gpu_shard_connect_local: engines must be unconnected ranks 0..world-1");
            if (e->lay.total != engines[0]->lay.total)
                throw std::invalid_argument("plnmf_gpu_shard_connect_local: ranks of different problems");
            one_device = one_device && e->device == engines[0]->device;
        }
        if (one_device && world > 1 && plnmf::lazy_module_loading())
            throw std::invalid_argument(
                "plnmf_gpu_shard_connect_local: ranks sharing one GPU need CUDA_MODULE_LOADING=EAGER "
                "(a lazily loaded kernel can wait for another rank's spinning kernel forever)");
        for (int g = 0; g < world; ++g) {
            plnmf_gpu_engine* e = engines[g];
            PLNMF_CUDA_CHECK(cudaSetDevice(e->device));
            for (int p = 0; p < world; ++p) {
                if (engines[p]->device != e->device) {
                    int ok = 0;
                    PLNMF_CUDA_CHECK(cudaDeviceCanAccessPeer(&ok, e->device, engines[p]->device));
                    if (!ok) throw plnmf::DeviceError("plnmf_gpu_shard_connect_local: no peer access between devices");
                    const cudaError_t r = cudaDeviceEnablePeerAccess(engines[p]->device, 0);
                    if (r == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else PLNMF_CUDA_CHECK(r);
                }
                e->peer_win[p] = engines[p]->win;
            }
            // ranks sharing one GPU: each persistent W kernel gets an equal share of the SMs so
            // that all ranks' kernels are resident together (they wait on one another)
            if (one_device && world > 1) e->sm_cap = e->sms / world;
            e->plan_tile = -1;
            e->have_ref_w = false;
            e->connected = true;
        }
    });
}

}  // extern "C"
