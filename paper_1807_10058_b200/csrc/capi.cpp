// C ABI of the B200 FCC-DCT (include/fcct_gpu.h). Host side: plan
// construction (plan.cpp), stage-table compilation for the fast pipeline,
// device uploads and kernel launches (kernels.cu). No exception crosses the
// ABI; failures map to fcct_status codes with a thread-local message.
#include <atomic>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fcct_gpu.h"
#include "kernels.hpp"
#include "orbit16.hpp"
#include "orbit_pat.hpp"
#include "orbit_big.hpp"
#include "host_stage.hpp"
#include "orbit_fft.hpp"
#include "plan.hpp"
#include "plan_cache.hpp"
#include "tiling.hpp"
#include "voxel_io.hpp"

namespace fcct {

const int* host_group_table() {
    static int table[24 * 9];
    static std::once_flag once;
    std::call_once(once, [] {
        const auto& g = s4_group();
        for (int e = 0; e < 24; ++e)
            for (int k = 0; k < 9; ++k) table[e * 9 + k] = g[e][k];
    });
    return table;
}

namespace {

thread_local std::string g_last_error;

struct CudaError : FcctError {
    explicit CudaError(const std::string& what, cudaError_t e)
        : FcctError(ST_CUDA, what + ": " + cudaGetErrorString(e)) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(what, e);
}

// ||D_n(p)||_1 for the plan-time condition estimate (plan.hpp ColNormHook): on
// the device of the plan being built (children may be derived on worker threads,
// whose current device is not the plan's).
std::atomic<int> g_colnorm_device{0};

double colnorm_on_device(int n, const Params& p) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return -1.0;  // no GPU: the host column sums
    }
    int prev = 0;
    ck(cudaGetDevice(&prev), "cudaGetDevice");
    const int dev = g_colnorm_device.load();
    if (dev != prev) ck(cudaSetDevice(dev), "cudaSetDevice");
    const int64_t N = cube(n);
    double* d = nullptr;
    cudaStream_t st = nullptr;
    std::vector<double> h(static_cast<size_t>(N));
    cudaError_t e = cudaMalloc(&d, sizeof(double) * N);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = dense_colnorm(n, p.r, p.s, p.t, d, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, sizeof(double) * N, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (st) cudaStreamDestroy(st);
    if (d) cudaFree(d);
    if (dev != prev) cudaSetDevice(prev);
    ck(e, "condition estimate (column norms)");
    return *std::max_element(h.begin(), h.end());
}

const bool g_colnorm_registered = [] {
    set_colnorm_hook(&colnorm_on_device);
    return true;
}();

// Tuning / debugging switches (stage masks, per-stage clocks, layout A/B runs)
// exist only in a library built with -DFCCT_AB_SWITCHES (tools/, never the
// product build): there no environment variable can change what a call computes.
const char* ab_env(const char* name) {
#ifdef FCCT_AB_SWITCHES
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

class DeviceGuard {
public:
    explicit DeviceGuard(int dev) {
        ck(cudaGetDevice(&prev_), "cudaGetDevice");
        if (prev_ != dev) {
            ck(cudaSetDevice(dev), "cudaSetDevice");
            switched_ = true;
        }
    }
    ~DeviceGuard() {  // nothing to restore on the caller's own device (a driver call per transform otherwise)
        if (switched_) cudaSetDevice(prev_);
    }

private:
    int prev_ = 0;
    bool switched_ = false;
};

// Device allocation owned by a plan.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t b) : bytes(b) { ck(cudaMalloc(&ptr, std::max<size_t>(b, 16)), "cudaMalloc"); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (ptr) cudaFree(ptr);
    }
};

template <typename T>
std::shared_ptr<DevBuf> upload(const std::vector<T>& v) {
    auto b = std::make_shared<DevBuf>(v.size() * sizeof(T));
    if (!v.empty()) ck(cudaMemcpy(b->ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return b;
}

// Row list of a sparse stage operator on the full n^3 vector.
struct Rows {
    int64_t N = 0;
    std::vector<std::vector<std::pair<int32_t, cld>>> r;
};

template <typename R>
void push_coef(std::vector<R>& out, const cld& v) {
    out.push_back(static_cast<R>(v.real()));
    out.push_back(static_cast<R>(v.imag()));
}

struct PipelineTables {
    PipelineDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
};

struct RootTables {
    RootDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
};

// Orbit-FFT executor (orbit_fft.hpp): register-resident base-change tiles.
struct OrbitFftTables {
    OrbitFftDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
    int64_t tiles = 0;
    double exec_flops = 0;
};

void upload_orbit_fft(const OrbitFftHost& h, OrbitFftTables& out) {
    out = OrbitFftTables{};
    auto bt = upload(h.table), bm = upload(h.meta), bn = upload(h.ntiles);
    out.bufs = {bt, bm, bn};
    OrbitFftDesc& d = out.desc;
    d.n = h.n;
    d.N = h.N;
    d.dir = h.dir;
    d.groups = h.groups;
    d.tmax = h.tmax;
    d.warps = h.warps;
    d.in_stride = d.out_stride = 0;
    d.table = static_cast<const double2*>(bt->ptr);
    d.meta = static_cast<const int2*>(bm->ptr);
    d.ntiles = static_cast<const int*>(bn->ptr);
    out.tiles = h.tiles;
    out.exec_flops = h.exec_flops();
}

// Two-pass orbit-FFT executor (n = 16, orbit16.hpp).
struct Orbit16Tables {
    Orbit16Desc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
    double exec_flops = 0;
};

void upload_orbit16(const Orbit16Host& h, Orbit16Tables& out) {
    out = Orbit16Tables{};
    auto bt = upload(h.table), bm = upload(h.tile_meta), bo = upload(h.out_pos), bg = upload(h.gather),
         bc = upload(h.chunk_slots), bz = upload(h.zperm);
    out.bufs = {bt, bm, bo, bg, bc, bz};
    Orbit16Desc& d = out.desc;
    d.n = h.n;
    d.N = h.N;
    d.dir = h.dir;
    d.nchunks = h.nchunks;
    d.tmax = h.tmax;
    d.table = static_cast<const double2*>(bt->ptr);
    d.tile_meta = static_cast<const int*>(bm->ptr);
    d.out_pos = static_cast<const int*>(bo->ptr);
    d.gather = static_cast<const int*>(bg->ptr);
    d.chunk_slots = static_cast<const int*>(bc->ptr);
    d.zperm = static_cast<const int*>(bz->ptr);
    out.exec_flops = h.exec_flops();
}

// Single-pass orbit-pattern executor (n = 16, orbit_pat.hpp).
struct OrbitPatTables {
    OrbitPatDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
    double exec_flops = 0, exec_flops_real = 0;
};

void upload_orbit_pat(const OrbitPatHost& h, OrbitPatTables& out) {
    out = OrbitPatTables{};
    OrbitPatDesc& d = out.desc;
    d.n = h.n;
    d.N = h.N;
    d.dir = h.dir;
    for (int c = 0; c < 2; ++c) {
        d.cnt[c] = h.cnt[c];
        d.ntiles[c] = h.ntiles[c];
        if (h.op[c].empty()) continue;
        auto bo = upload(h.op[c]);
        out.bufs.push_back(bo);
        d.op[c] = static_cast<const double2*>(bo->ptr);
    }
    auto narrow = [](const std::vector<int32_t>& v) { return std::vector<uint16_t>(v.begin(), v.end()); };
    auto bi = upload(narrow(h.idx)), bw = upload(h.warp_tiles);
    out.bufs.insert(out.bufs.end(), {bi, bw});
    d.idx = static_cast<const uint16_t*>(bi->ptr);
    d.idx_count = static_cast<int>(h.idx.size());
    d.warp_tiles = static_cast<const int2*>(bw->ptr);
    d.nrare = h.nrare;
    d.rare_pitch = h.rare_pitch;
    for (int ax = 0; ax < 3; ++ax)
        for (int x = 0; x < 16; ++x) d.lax[ax][x] = make_double2(h.lax[ax][x][0], h.lax[ax][x][1]);
    if (d.nrare > 0) {
        auto br = upload(narrow(h.rare_out)), bn = upload(narrow(h.rare_in)), bc = upload(h.rare_coef);
        out.bufs.insert(out.bufs.end(), {br, bn, bc});
        d.rare_out = static_cast<const uint16_t*>(br->ptr);
        d.rare_in = static_cast<const uint16_t*>(bn->ptr);
        d.rare_coef = static_cast<const double2*>(bc->ptr);
    }
    out.exec_flops = h.exec_flops();
    out.exec_flops_real = h.exec_flops(true);
}

// Large-n S pass on the orbit-pattern tables (n = 32, 64, orbit_pat.hpp).
struct OrbitPatBigTables {
    OrbitPatBigDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
    double exec_flops = 0;
};

void upload_orbit_pat_big(const OrbitPatHost& h, OrbitPatBigTables& out) {
    out = OrbitPatBigTables{};
    OrbitPatBigDesc& d = out.desc;
    d.n = h.n;
    d.N = h.N;
    d.dir = h.dir;
    while ((1 << d.log2n) < h.n) ++d.log2n;
    for (int c = 0; c < 2; ++c) {
        d.cnt[c] = h.cnt[c];
        d.ntiles[c] = h.ntiles[c];
        if (h.op[c].empty()) continue;
        auto bo = upload(h.op[c]);
        out.bufs.push_back(bo);
        d.op[c] = static_cast<const double2*>(bo->ptr);
    }
    std::vector<double> lax(static_cast<size_t>(3) * h.n * 2);
    for (int ax = 0; ax < 3; ++ax)
        for (int x = 0; x < h.n; ++x) {
            lax[(static_cast<size_t>(ax) * h.n + x) * 2] = h.lax[ax][x][0];
            lax[(static_cast<size_t>(ax) * h.n + x) * 2 + 1] = h.lax[ax][x][1];
        }
    auto bi = upload(h.idx), bl = upload(lax);
    out.bufs.insert(out.bufs.end(), {bi, bl});
    d.idx = static_cast<const int32_t*>(bi->ptr);
    d.lax = static_cast<const double2*>(bl->ptr);
    d.nrare = h.nrare;
    d.rare_pitch = h.rare_pitch;
    if (d.nrare > 0) {
        auto br = upload(h.rare_out), bn = upload(h.rare_in), bc = upload(h.rare_coef);
        out.bufs.insert(out.bufs.end(), {br, bn, bc});
        d.rare_out = static_cast<const int32_t*>(br->ptr);
        d.rare_in = static_cast<const int32_t*>(bn->ptr);
        d.rare_coef = static_cast<const double2*>(bc->ptr);
    }
    out.exec_flops = h.exec_flops();
}

// Large-n orbit-FFT executor (n = 32, 64, orbit_big.hpp).
struct OrbitBigTables {
    OrbitBigDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
    double exec_flops = 0;
};

void upload_orbit_big(const OrbitBigHost& h, OrbitBigTables& out) {
    out = OrbitBigTables{};
    auto b1 = upload(h.row_orbit), b2 = upload(h.row_index), b3 = upload(h.orbit_off), b4 = upload(h.coef_off),
         b5 = upload(h.members), b6 = upload(h.coef);
    out.bufs = {b1, b2, b3, b4, b5, b6};
    OrbitBigDesc& d = out.desc;
    d.n = h.n;
    d.N = h.N;
    d.dir = h.dir;
    d.rows = h.N;
    d.row_orbit = static_cast<const int*>(b1->ptr);
    d.row_index = static_cast<const int*>(b2->ptr);
    d.orbit_off = static_cast<const int*>(b3->ptr);
    d.coef_off = static_cast<const int64_t*>(b4->ptr);
    d.members = static_cast<const int*>(b5->ptr);
    d.coef = static_cast<const double2*>(b6->ptr);
    if (h.gen) {
        // (mpack, the per-slot packing, is the host emulation's view; the kernel reads fpack / tail)
        auto g2 = upload(h.ttab), g3 = upload(h.mtab), g4 = upload(h.grp), g5 = upload(h.fpack), g6 = upload(h.tail),
             g7 = upload(h.fbase);
        out.bufs.insert(out.bufs.end(), {g2, g3, g4, g5, g6, g7});
        d.fbase = static_cast<const double2*>(g7->ptr);
        d.fpack = static_cast<const uint32_t*>(g5->ptr);
        d.nfree = static_cast<int>(h.fpack.size() / 24);
        d.tail = static_cast<const int*>(g6->ptr);
        d.ntail = static_cast<int>(h.tail.size());
        d.gen = 1;
        d.pr = h.pr;
        d.ps = h.ps;
        d.pt = h.pt;
        d.ttab = static_cast<const double2*>(g2->ptr);
        d.mtab = static_cast<const uint8_t*>(g3->ptr);
        d.grp = static_cast<const int*>(g4->ptr);
        d.ncarry = h.ncarry;
    }
    out.exec_flops = h.exec_flops();
}

struct Pipeline2Tables {
    Pipeline2Desc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
    int64_t dmma_per_tile = 0;
};

void upload_pipeline2(const Pipeline2Host& h, Pipeline2Tables& out) {
    out.desc = Pipeline2Desc{};
    out.desc.tb = h.shape.tb;
    out.desc.warps = h.shape.warps;
    out.desc.N = h.N;
    out.desc.stride = h.stride;
    out.desc.row_in = out.desc.row_out = 2 * static_cast<int64_t>(h.N);
    out.desc.nstages = static_cast<int>(h.stages.size());
    const char* ds = ab_env("FCCT_DIRECT_STORE");
    out.desc.direct_store = ds ? std::atoi(ds) : 0;
    const char* sm = ab_env("FCCT_DEBUG_STAGE_MASK");  // timing experiments only
    out.desc.stage_mask = sm ? std::atoi(sm) : -1;
    out.desc.ring = 1;  // sparse-stage table entries stream through the per-warp cp.async ring
    out.desc.timing = nullptr;
    if (ab_env("FCCT_DEBUG_TIMING")) {  // per-stage clock64 totals of CTA 0 (profiling aid)
        auto b = std::make_shared<DevBuf>(sizeof(unsigned long long) * (kMaxStages + 2 + kMaxStages * 16));
        ck(cudaMemset(b->ptr, 0, b->bytes), "memset");
        out.desc.timing = static_cast<unsigned long long*>(b->ptr);
        out.bufs.push_back(b);
    }
    out.dmma_per_tile = h.dmma_per_tile;
    if (out.desc.nstages > kMaxStages) throw FcctError(ST_INVALID_ARGUMENT, "too many stages");
    std::vector<unsigned char> arena;
    auto put = [&](const void* data, size_t bytes) -> int {
        if (bytes == 0) return -1;
        const size_t off = (arena.size() + 15) & ~size_t{15};
        arena.resize(off + bytes);
        std::memcpy(arena.data() + off, data, bytes);
        return static_cast<int>(off);
    };
    auto keep = [&](std::shared_ptr<DevBuf> b) {
        out.bufs.push_back(b);
        return b->ptr;
    };
    constexpr size_t kArenaK = 16 * 1024;  // K tables up to this size go to shared memory
    const char* gs = ab_env("FCCT_V2_GROUP_SYNC");  // A/B switch: 0 = CTA-wide barriers only
    const bool group_sync = gs ? std::atoi(gs) != 0 : true;
    const char* ns = ab_env("FCCT_V2_NAT_SHIFT");  // A/B switch: 0 = unshifted natural rows
    const bool nat_shift = ns ? std::atoi(ns) != 0 : true;
    out.desc.shift_in = nat_shift ? 2 * h.shift_in : 0;
    out.desc.shift_out = nat_shift ? 2 * h.shift_out : 0;
    for (size_t s = 0; s < h.stages.size(); ++s) {
        const Stage2Host& st = h.stages[s];
        Stage2Dev& d = out.desc.st[s];
        d = Stage2Dev{};
        d.kind = st.kind;
        d.n_units = st.n_units;
        d.sync_mid = group_sync ? st.sync_mid : 0;
        d.sync_end = group_sync ? st.sync_end : 0;
        d.ld_shift = (s == 0 && nat_shift) ? 16 * h.shift_in : 0;
        d.st_shift = (s + 1 == h.stages.size() && nat_shift) ? 16 * h.shift_out : 0;
        d.o_warp_units = put(st.warp_units.data(), st.warp_units.size() * 4);
        d.o_u_out = put(st.u_out.data(), st.u_out.size() * 4);
        d.o_w_base = d.o_w_count = d.o_w_ccount = d.o_e_slots = d.o_u_node = d.o_u_in = d.o_K = -1;
        if (st.kind == 0) {
            d.o_w_base = put(st.w_base.data(), st.w_base.size() * 4);
            d.o_w_count = put(st.w_count.data(), st.w_count.size() * 4);
            d.o_w_ccount = put(st.w_ccount.data(), st.w_ccount.size() * 4);
            d.o_e_slots = put(st.e_slots.data(), st.e_slots.size() * 4);
            d.e_re = static_cast<const double*>(keep(upload(st.e_re)));
            d.e_im = static_cast<const double*>(keep(upload(st.e_im)));
            std::vector<double> ri(2 * st.e_re.size());
            for (size_t q = 0; q < st.e_re.size(); ++q) {
                ri[2 * q] = st.e_re[q];
                ri[2 * q + 1] = st.e_im[q];
            }
            d.e_ri = static_cast<const double2*>(keep(upload(ri)));
        } else {
            d.o_u_node = put(st.u_node.data(), st.u_node.size() * 4);
            d.o_u_in = put(st.u_in.data(), st.u_in.size() * 4);
            d.K = static_cast<const double2*>(keep(upload(st.K)));
            if (st.K.size() * sizeof(double) <= kArenaK) d.o_K = put(st.K.data(), st.K.size() * sizeof(double));
        }
    }
    arena.resize((arena.size() + 15) & ~size_t{15});
    out.desc.arena_bytes = static_cast<int>(arena.size());
    out.desc.arena = static_cast<const uint4*>(keep(upload(arena)));
}

// ELL packing of a sparse stage for row groups of RG rows.
template <typename R>
void add_sparse_stage(PipelineTables& pt, const Rows& rows, int RG, const std::vector<int32_t>* gather,
                      const std::vector<int32_t>* scatter) {
    const int64_t N = rows.N;
    std::vector<int32_t> order(N);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return rows.r[a].size() > rows.r[b].size(); });
    const int64_t ngroups = (N + RG - 1) / RG;
    std::vector<int2> ginfo(ngroups);
    std::vector<int32_t> grow(ngroups * RG, -1), ecol;
    std::vector<R> ecoef;
    for (int64_t g = 0; g < ngroups; ++g) {
        int kmax = 0;
        for (int rr = 0; rr < RG; ++rr) {
            const int64_t idx = g * RG + rr;
            if (idx < N) kmax = std::max<int>(kmax, static_cast<int>(rows.r[order[idx]].size()));
        }
        ginfo[g] = make_int2(static_cast<int>(ecol.size()), kmax);
        for (int k = 0; k < kmax; ++k)
            for (int rr = 0; rr < RG; ++rr) {
                const int64_t idx = g * RG + rr;
                if (idx < N && k < static_cast<int>(rows.r[order[idx]].size())) {
                    const auto& e = rows.r[order[idx]][k];
                    ecol.push_back(gather ? (*gather)[e.first] : e.first);
                    push_coef(ecoef, e.second);
                } else {
                    ecol.push_back(0);
                    push_coef(ecoef, cld{0, 0});
                }
            }
        for (int rr = 0; rr < RG; ++rr) {
            const int64_t idx = g * RG + rr;
            if (idx < N) grow[g * RG + rr] = scatter ? (*scatter)[order[idx]] : order[idx];
        }
    }
    auto b_ginfo = upload(ginfo), b_grow = upload(grow), b_ecol = upload(ecol), b_ecoef = upload(ecoef);
    StageDesc& sd = pt.desc.stage[pt.desc.nstages++];
    sd = StageDesc{};
    sd.kind = 0;
    sd.ngroups = static_cast<int>(ngroups);
    sd.ginfo = static_cast<const int2*>(b_ginfo->ptr);
    sd.grow = static_cast<const int*>(b_grow->ptr);
    sd.ecol = static_cast<const int*>(b_ecol->ptr);
    sd.ecoef = b_ecoef->ptr;
    pt.bufs.insert(pt.bufs.end(), {b_ginfo, b_grow, b_ecol, b_ecoef});
}

template <typename R>
void add_mix_stage(PipelineTables& pt, const std::vector<const PlanNode*>& nodes, bool inverse,
                   const std::vector<int32_t>* gather, const std::vector<int32_t>* scatter) {
    std::vector<R> K;
    for (const PlanNode* nd : nodes)
        for (int i = 0; i < 64; ++i) push_coef(K, inverse ? nd->Kinv[i] : nd->K[i]);
    auto bK = upload(K);
    StageDesc& sd = pt.desc.stage[pt.desc.nstages++];
    sd = StageDesc{};
    sd.kind = 1;
    sd.nodes = static_cast<int>(nodes.size());
    sd.m3 = static_cast<int>(cube(nodes[0]->n / 2));
    sd.K = bK->ptr;
    pt.bufs.push_back(bK);
    if (gather) {
        auto b = upload(*gather);
        sd.gather = static_cast<const int*>(b->ptr);
        pt.bufs.push_back(b);
    }
    if (scatter) {
        auto b = upload(*scatter);
        sd.scatter = static_cast<const int*>(b->ptr);
        pt.bufs.push_back(b);
    }
}

// Block-diagonal sparse operator over the nodes of one level.
Rows level_rows(const std::vector<const PlanNode*>& nodes, int kind /*0 B, 1 Binv, 2 D, 3 Dinv*/) {
    Rows rows;
    const int64_t s3 = cube(nodes[0]->n);
    rows.N = s3 * static_cast<int64_t>(nodes.size());
    rows.r.resize(rows.N);
    for (size_t q = 0; q < nodes.size(); ++q) {
        const PlanNode& nd = *nodes[q];
        const int64_t off = static_cast<int64_t>(q) * s3;
        if (kind <= 1) {
            const SparseLD& S = kind == 0 ? nd.B : nd.Binv;
            for (int64_t r = 0; r < s3; ++r)
                for (int64_t k = S.rowptr[r]; k < S.rowptr[r + 1]; ++k)
                    rows.r[off + r].emplace_back(static_cast<int32_t>(off + S.col[k]), S.val[k]);
        } else {
            const auto& M = kind == 2 ? nd.D : nd.Dinv;
            for (int64_t r = 0; r < s3; ++r)
                for (int64_t c = 0; c < s3; ++c)
                    rows.r[off + r].emplace_back(static_cast<int32_t>(off + c), M[r * s3 + c]);
        }
    }
    return rows;
}

std::vector<int32_t> composite_order(const PlanNode& nd) {
    // Z_s(i) = perm_s[blk*m^3 + Z_m(j)] for radix nodes, identity for direct.
    const int64_t s3 = cube(nd.n);
    std::vector<int32_t> z(s3);
    if (!nd.radix) {
        std::iota(z.begin(), z.end(), 0);
        return z;
    }
    const auto sub = composite_order(*nd.children[0]);
    const auto perm = radix_permutation(nd.n);
    const int64_t m3 = s3 / 8;
    for (int64_t i = 0; i < s3; ++i) z[i] = static_cast<int32_t>(perm[(i / m3) * m3 + sub[i % m3]]);
    return z;
}

int choose_tb(int64_t N, bool f32) {
    const int64_t row_bytes = (N + (f32 ? 2 : 1)) * (f32 ? 8 : 16);
    for (int tb : {32, 16, 8, 4, 2, 1})
        if (N * tb <= 8192 && 128 + tb * row_bytes <= 227 * 1024) return tb;
    return 0;
}

template <typename R>
void build_pipelines(const PlanNode& root, int tb, PipelineTables& fwd, PipelineTables& inv) {
    const int RG = 32 / tb;
    std::vector<std::vector<const PlanNode*>> levels;
    std::vector<const PlanNode*> cur{&root};
    while (!cur.empty() && cur[0]->radix) {
        levels.push_back(cur);
        std::vector<const PlanNode*> next;
        for (const PlanNode* nd : cur)
            for (const auto& c : nd->children) next.push_back(c.get());
        cur = next;
    }
    const std::vector<const PlanNode*> leaves = cur;  // direct nodes
    const bool dense_leaves = leaves[0]->n > 1;
    const auto Z = composite_order(root);
    for (auto* pt : {&fwd, &inv}) {
        pt->desc.n = root.n;
        pt->desc.N = static_cast<int>(cube(root.n));
        pt->desc.tb = tb;
        pt->desc.nstages = 0;
    }
    // forward: for each level B (size > 2) then K-mix; dense leaves last.
    const int nfwd = [&] {
        int c = 0;
        for (auto& lv : levels) c += (level_identity(lv, false) ? 1 : 2);
        return c + (dense_leaves ? 1 : 0);
    }();
    int s = 0;
    for (auto& lv : levels) {
        if (!level_identity(lv, false)) {
            add_sparse_stage<R>(fwd, level_rows(lv, 0), RG, nullptr, (++s == nfwd) ? &Z : nullptr);
        }
        add_mix_stage<R>(fwd, lv, false, nullptr, (++s == nfwd) ? &Z : nullptr);
    }
    if (dense_leaves) add_sparse_stage<R>(fwd, level_rows(leaves, 2), RG, nullptr, &Z);
    // inverse: dense leaves first, then per level (deepest first) K^{-1} mix then B^{-1}.
    bool first = true;
    if (dense_leaves) {
        add_sparse_stage<R>(inv, level_rows(leaves, 3), RG, &Z, nullptr);
        first = false;
    }
    for (auto it = levels.rbegin(); it != levels.rend(); ++it) {
        add_mix_stage<R>(inv, *it, true, first ? &Z : nullptr, nullptr);
        first = false;
        if (!level_identity(*it, true)) add_sparse_stage<R>(inv, level_rows(*it, 1), RG, nullptr, nullptr);
    }
}

struct GlobalTables {
    GlobalPipelineDesc desc{};
    std::vector<std::shared_ptr<DevBuf>> bufs;
};

template <typename R>
void add_global_sparse(GlobalTables& gt, const Rows& rows, const std::vector<int32_t>* gather,
                       const std::vector<int32_t>* scatter) {
    // sliced ELL: rows sorted by length (the output position map absorbs the
    // order), slices of 32 rows padded to their longest row, entries stored
    // [slice][e][lane] so every warp-wide table load is one contiguous 512 B
    // (complex128) run
    const int64_t N = rows.N;
    std::vector<int32_t> order(N);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return rows.r[a].size() > rows.r[b].size(); });
    const int64_t nslices = (N + 31) / 32;
    std::vector<int64_t> slice_off(nslices + 1, 0);
    for (int64_t sl = 0; sl < nslices; ++sl) {
        size_t w = 0;
        for (int64_t l = 0; l < 32 && sl * 32 + l < N; ++l) w = std::max(w, rows.r[order[sl * 32 + l]].size());
        slice_off[sl + 1] = slice_off[sl] + static_cast<int64_t>(w) * 32;
    }
    std::vector<int32_t> col(slice_off[nslices], 0);
    std::vector<R> coef(2 * slice_off[nslices], R(0));
    std::vector<int32_t> out_row(N);
    for (int64_t i = 0; i < N; ++i) {
        const int64_t sl = i / 32, lane = i % 32;
        const auto& row = rows.r[order[i]];
        for (size_t e = 0; e < row.size(); ++e) {
            const int64_t idx = slice_off[sl] + static_cast<int64_t>(e) * 32 + lane;
            col[idx] = gather ? (*gather)[row[e].first] : row[e].first;
            std::vector<R> c;
            push_coef(c, row[e].second);
            coef[2 * idx] = c[0];
            coef[2 * idx + 1] = c[1];
        }
        out_row[i] = scatter ? (*scatter)[order[i]] : order[i];
    }
    GStage& st = gt.desc.st[gt.desc.nstages++];
    st = GStage{};
    st.kind = 0;
    auto b1 = upload(slice_off), b2 = upload(col), b3 = upload(coef), b4 = upload(out_row);
    st.rowptr = static_cast<const int64_t*>(b1->ptr);
    st.col = static_cast<const int*>(b2->ptr);
    st.coef = b3->ptr;
    st.out_row = static_cast<const int*>(b4->ptr);
    gt.bufs.insert(gt.bufs.end(), {b1, b2, b3, b4});
}

template <typename R>
void add_global_mix(GlobalTables& gt, const std::vector<const PlanNode*>& nodes, bool inverse,
                    const std::vector<int32_t>* gather, const std::vector<int32_t>* scatter) {
    std::vector<R> K;
    for (const PlanNode* nd : nodes)
        for (int i = 0; i < 64; ++i) push_coef(K, inverse ? nd->Kinv[i] : nd->K[i]);
    GStage& st = gt.desc.st[gt.desc.nstages++];
    st = GStage{};
    st.kind = 1;
    st.nodes = static_cast<int>(nodes.size());
    st.m3 = static_cast<int>(cube(nodes[0]->n / 2));
    auto bK = upload(K);
    st.K = bK->ptr;
    gt.bufs.push_back(bK);
    if (gather) {
        auto b = upload(*gather);
        st.gather = static_cast<const int*>(b->ptr);
        gt.bufs.push_back(b);
    }
    if (scatter) {
        auto b = upload(*scatter);
        st.scatter = static_cast<const int*>(b->ptr);
        gt.bufs.push_back(b);
    }
}

// Stage lists of the global multi-pass pipeline (same order as build_pipelines).
template <typename R>
void build_global_pipelines(const PlanNode& root, GlobalTables& fwd, GlobalTables& inv) {
    std::vector<std::vector<const PlanNode*>> levels;
    std::vector<const PlanNode*> cur{&root};
    while (!cur.empty() && cur[0]->radix) {
        levels.push_back(cur);
        std::vector<const PlanNode*> next;
        for (const PlanNode* nd : cur)
            for (const auto& c : nd->children) next.push_back(c.get());
        cur = next;
    }
    const std::vector<const PlanNode*> leaves = cur;
    const bool dense_leaves = leaves[0]->n > 1;
    const auto Z = composite_order(root);
    for (auto* gt : {&fwd, &inv}) {
        gt->desc.N = static_cast<int>(cube(root.n));
        gt->desc.nstages = 0;
    }
    int nfwd = dense_leaves ? 1 : 0;
    for (auto& lv : levels) nfwd += level_identity(lv, false) ? 1 : 2;
    if (nfwd > kMaxStages) throw FcctError(ST_INVALID_ARGUMENT, "too many stages");
    int s = 0;
    for (auto& lv : levels) {
        if (!level_identity(lv, false)) add_global_sparse<R>(fwd, level_rows(lv, 0), nullptr, (++s == nfwd) ? &Z : nullptr);
        add_global_mix<R>(fwd, lv, false, nullptr, (++s == nfwd) ? &Z : nullptr);
    }
    if (dense_leaves) add_global_sparse<R>(fwd, level_rows(leaves, 2), nullptr, &Z);
    bool first = true;
    if (dense_leaves) {
        add_global_sparse<R>(inv, level_rows(leaves, 3), &Z, nullptr);
        first = false;
    }
    for (auto it = levels.rbegin(); it != levels.rend(); ++it) {
        add_global_mix<R>(inv, *it, true, first ? &Z : nullptr, nullptr);
        first = false;
        if (!level_identity(*it, true)) add_global_sparse<R>(inv, level_rows(*it, 1), nullptr, nullptr);
    }
}

}  // namespace
}  // namespace fcct

using namespace fcct;

struct fcct_plan_s {
    int n = 0;
    Params p;
    int method = FCCT_FAST;
    int precision = FCCT_F64;
    int device = 0;
    int num_sms = 148;
    bool radix = false;
    std::shared_ptr<const PlanNode> tree;
    bool tree_exact = false;  // built here by build_tree: the exact factorisation by construction
    PipelineTables fwd, inv;
    bool offt = false;  // orbit-FFT executor (telescoped radix tree, orbit_fft.hpp)
    OrbitFftTables ofwd, ofinv;
    bool o16 = false;  // two-pass orbit-FFT executor (n = 16, orbit16.hpp)
    Orbit16Tables o16fwd, o16inv;
    bool opat = false;  // single-pass orbit-pattern executor (n = 16, orbit_pat.hpp)
    OrbitPatTables opfwd, opinv;
    bool obig = false;  // large-n orbit-FFT executor (n = 32, 64, fp64, orbit_big.hpp)
    OrbitBigTables obfwd, obinv;
    bool obpat = false;  // ... its S pass on the orbit-pattern tables (constant operator in registers)
    OrbitPatBigTables obpfwd, obpinv;
    bool v2 = false;  // fp64 DMMA pipeline (tiling.hpp)
    Pipeline2Tables fwd2, inv2;
    bool two_level = false;  // n = 16: root pass + eight n = 8 child pipelines
    RootTables rfwd, rinv;
    Pipeline2Tables cfwd[8], cinv[8];
    bool child_offt = false;  // the eight n = 8 children run on the orbit-FFT executor
    OrbitFftTables ocfwd[8], ocinv[8];
    cudaStream_t cs[4] = {nullptr, nullptr, nullptr, nullptr};  // child pipelines run concurrently
    cudaEvent_t cev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    bool global = false;  // global-memory multi-pass pipeline
    GlobalTables gfwd, ginv;
    std::shared_ptr<DevBuf> scratch0, scratch1;
    int exec_force = 0;  // fcct_executor requested at creation (FCCT_EXEC_AUTO = the default choice)
    std::mutex scratch_mu;
    // stream-ordered ownership of the scratch: recorded after the last kernel
    // of a call that used it; the next call's stream waits on it (no host sync)
    cudaEvent_t scratch_ev = nullptr;
    std::shared_ptr<DevBuf> Wt_fwd, Wt_inv;
    std::shared_ptr<DevBuf> Wt_fwd_lo, Wt_inv_lo;  // tcgen05 3xTF32 plans: Wt_* hold the rna_tf32 parts
    bool tc32 = false;                              // fp32 direct plan on tcgen05 (gemm_tc.cu)
    // fp64 direct plans on tcgen05 (Ozaki int8 slices): W slices + row scales per direction,
    // and a per-call workspace for the slices of the input batch
    bool oz64 = false;
    std::shared_ptr<DevBuf> oz_w[2], oz_ws[2];
    std::shared_ptr<DevBuf> oz_in, oz_in_scale;
    std::vector<std::shared_ptr<DevBuf>> extra;
    fcct_plan_info_t info{};
    // workspace for host-buffer calls and in-place direct calls
    std::mutex ws_mu;
    std::shared_ptr<DevBuf> ws_in[2], ws_out[2];
    cudaStream_t hs[2] = {nullptr, nullptr};  // host-path copy/compute streams
    cudaEvent_t hev = nullptr;
    // pinned bounce buffers for pageable host buffers (host_stage.hpp)
    PinnedBuf pin_in[2], pin_out[2];
    cudaEvent_t h2d_ev[2] = {nullptr, nullptr}, d2h_ev[2] = {nullptr, nullptr};
    ~fcct_plan_s() {
        for (auto e : h2d_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : d2h_ev)
            if (e) cudaEventDestroy(e);
        for (auto& h : hs)
            if (h) cudaStreamDestroy(h);
        for (auto& h : cs)
            if (h) cudaStreamDestroy(h);
        for (auto& e : cev)
            if (e) cudaEventDestroy(e);
        if (hev) cudaEventDestroy(hev);
        if (scratch_ev) cudaEventDestroy(scratch_ev);
    }
    // complex staging for real-I/O calls on executors without fused real I/O
    std::mutex ws_real_mu;
    std::shared_ptr<DevBuf> ws_real;
};

namespace {

int64_t elem_bytes(const fcct_plan_s* p) { return p->precision == FCCT_F32 ? 8 : 16; }

// The plan-owned scratch (z / ping-pong buffers) is shared by every call on the
// plan: a call holds scratch_mu while it enqueues, makes its stream wait for
// the previous user's last kernel, and records its own last kernel. Calls on
// one stream stay asynchronous; calls on different streams are ordered on the
// device, not by blocking the host.
void scratch_acquire(fcct_plan_s* pl, cudaStream_t st) {
    if (!pl->scratch_ev)
        ck(cudaEventCreateWithFlags(&pl->scratch_ev, cudaEventDisableTiming), "event");
    else
        ck(cudaStreamWaitEvent(st, pl->scratch_ev, 0), "scratch wait");
}
void scratch_release(fcct_plan_s* pl, cudaStream_t st) { ck(cudaEventRecord(pl->scratch_ev, st), "scratch record"); }
// Before a scratch buffer is replaced (and freed): wait for its last user, which
// may be a call on another stream (scratch_ev), as well as this stream's work.
void scratch_retire(fcct_plan_s* pl, cudaStream_t st) {
    ck(cudaStreamSynchronize(st), "sync");
    if (pl->scratch_ev) ck(cudaEventSynchronize(pl->scratch_ev), "scratch event sync");
}

// Ozaki slice counts: the inverse's error is amplified by the conditioning of
// D^{-1}, so it carries one more slice (fp64-level accuracy, tools/ozaki_sim.py)
constexpr int kOzaki_forward = 7, kOzaki_inverse = 8;

void build_direct(fcct_plan_s* pl) {
    const int n = pl->n;
    const int64_t N = cube(n);
    const bool f32 = pl->precision == FCCT_F32;
    const size_t wbytes = static_cast<size_t>(2 * N) * (2 * N) * (f32 ? 4 : 8);
    // fp32 plans whose real form tiles by 128 run on tcgen05 (3xTF32): the tables
    // are generated in fp64 and split into (W_hi, W_lo)
    pl->tc32 = f32 && gemm_tf32x3_supported(static_cast<int>(2 * N), static_cast<int>(2 * N));
    const size_t count = static_cast<size_t>(2 * N) * (2 * N);
    std::shared_ptr<DevBuf> w64;
    if (pl->tc32) w64 = std::make_shared<DevBuf>(count * 8);
    pl->Wt_fwd = std::make_shared<DevBuf>(wbytes);
    pl->Wt_inv = std::make_shared<DevBuf>(wbytes);
    if (pl->tc32) {
        pl->Wt_fwd_lo = std::make_shared<DevBuf>(wbytes);
        pl->Wt_inv_lo = std::make_shared<DevBuf>(wbytes);
        ck(gen_dense_realform(n, pl->p.r, pl->p.s, pl->p.t, w64->ptr, false, nullptr), "gen_dense_realform");
        ck(split_tf32(static_cast<const double*>(w64->ptr), static_cast<float*>(pl->Wt_fwd->ptr),
                      static_cast<float*>(pl->Wt_fwd_lo->ptr), static_cast<int64_t>(count), nullptr),
           "split_tf32");
    } else {
        ck(gen_dense_realform(n, pl->p.r, pl->p.s, pl->p.t, pl->Wt_fwd->ptr, f32, nullptr), "gen_dense_realform");
    }
    // orbit blocks of S_n(p)^{-1} -> device, then D^{-1} generated on the device
    OrbitBlocks ob = orbit_blocks(n, pl->p);
    if (!std::isfinite(ob.worst_condition))
        throw FcctError(ST_ILL_CONDITIONED, "dense transform: condition estimate inf exceeds 1e12");
    const Orbits& orb = *ob.orb;
    std::vector<int32_t> mem_off{0}, mem, sinv_off;
    std::vector<double> sinv;
    for (size_t o = 0; o < orb.members.size(); ++o) {
        sinv_off.push_back(static_cast<int32_t>(sinv.size() / 2));
        for (int32_t a : orb.members[o]) mem.push_back(a);
        mem_off.push_back(static_cast<int32_t>(mem.size()));
        for (const cld& v : ob.Sinv[o]) {
            sinv.push_back(static_cast<double>(v.real()));
            sinv.push_back(static_cast<double>(v.imag()));
        }
    }
    auto b1 = upload(orb.orbit_of), b2 = upload(orb.pos), b3 = upload(mem_off), b4 = upload(mem),
         b5 = upload(sinv_off), b6 = upload(sinv);
    OrbitDev od{static_cast<const int*>(b1->ptr), static_cast<const int*>(b2->ptr),
                static_cast<const int*>(b3->ptr), static_cast<const int*>(b4->ptr),
                static_cast<const int*>(b5->ptr), static_cast<const double*>(b6->ptr)};
    if (pl->tc32) {
        ck(gen_dense_inv_realform(n, od, w64->ptr, false, nullptr), "gen_dense_inv_realform");
        ck(split_tf32(static_cast<const double*>(w64->ptr), static_cast<float*>(pl->Wt_inv->ptr),
                      static_cast<float*>(pl->Wt_inv_lo->ptr), static_cast<int64_t>(count), nullptr),
           "split_tf32");
    } else {
        ck(gen_dense_inv_realform(n, od, pl->Wt_inv->ptr, f32, nullptr), "gen_dense_inv_realform");
    }
    // fp64 plans whose real form tiles by 64 (n = 4, 8, 16) run on tcgen05 by the
    // Ozaki scheme: int8 slices of D / D^{-1} (real form, rows = outputs) with row scales
    pl->oz64 = !f32 && gemm_ozaki_supported(static_cast<int>(2 * N), static_cast<int>(2 * N));
    if (pl->oz64) {
        const int K = static_cast<int>(2 * N);
        for (int dir = 0; dir < 2; ++dir) {
            const int S = dir ? kOzaki_inverse : kOzaki_forward;
            pl->oz_w[dir] = std::make_shared<DevBuf>(static_cast<size_t>(S) * K * K);
            pl->oz_ws[dir] = std::make_shared<DevBuf>(static_cast<size_t>(K) * 8);
            ck(ozaki_slice(static_cast<const double*>((dir ? pl->Wt_inv : pl->Wt_fwd)->ptr), K, K, S,
                           static_cast<int8_t*>(pl->oz_w[dir]->ptr), static_cast<double*>(pl->oz_ws[dir]->ptr),
                           nullptr),
               "ozaki slices");
        }
    }
    ck(cudaDeviceSynchronize(), "direct table generation");
    // the reference's estimate and gate (assemble_direct: condition_with_lu(D),
    // transform.cpp:339-344; dense_transform stores it for n^3 <= 512, :141-142)
    pl->info.condition = reference_condition(n, pl->p);
    if (!(pl->info.condition <= 1e12))
        throw FcctError(ST_ILL_CONDITIONED, "dense transform (n=" + std::to_string(n) + "): condition estimate " +
                                                std::to_string(pl->info.condition) + " exceeds 1e12");
    pl->info.table_bytes = static_cast<int64_t>((pl->tc32 ? 4 : 2) * wbytes);
}

void build_v2(fcct_plan_s* pl) {
    pl->v2 = false;
    if (pl->exec_force == FCCT_EXEC_TILE) return;
    Shape2 shape;  // default: 16 blocks x 16 warps, one CTA per SM
    if (const char* sh = ab_env("FCCT_V2_SHAPE"); sh && std::string(sh) == "8x8")
        shape = Shape2{8, 8, 8};  // two CTAs per SM (tuning experiment)
    Pipeline2Host hf, hi;
    if (!compile_pipeline2(*pl->tree, false, shape, hf) || !compile_pipeline2(*pl->tree, true, shape, hi)) return;
    upload_pipeline2(hf, pl->fwd2);
    upload_pipeline2(hi, pl->inv2);
    // fp32 plans: complex64 in HBM, fp64 arithmetic in the tile (the FP64 tensor
    // pipe has no fp32 kind; TF32 would miss the 1e-5 bar)
    pl->fwd2.desc.io_f32 = pl->inv2.desc.io_f32 = pl->precision == FCCT_F32 ? 1 : 0;
    if (pl->fwd2.desc.io_f32) pl->fwd2.desc.direct_store = pl->inv2.desc.direct_store = 0;
    pl->v2 = true;
}

// Two-level executor (n = 16): the root B and K run as one SIMT pass over a
// child-major scratch, the eight n = 8 children on the DMMA pipeline (each
// reading and writing its 512-point slice of every block), and one gather
// applies the radix permutation. Inverse: gather, children, root pass.
// ELL layout of the root-level rows, 8 groups g of m3 rows g m3 + h (thread h
// handles row g m3 + h of every group). Within each warp's 32 rows the entries
// of every step are reordered so the 8 lanes of each quarter-warp gather
// x[col] from distinct 16-byte bank groups (col mod 8) where possible; padding
// entries (value 0) take a free bank group too.
void build_root_ell(const SparseLD& S, int N, RootTables& rt, RootDesc& d) {
    const int m3 = N / 8;
    std::vector<int> width(8, 0);
    for (int g = 0; g < 8; ++g)
        for (int h = 0; h < m3; ++h) {
            const int64_t row = static_cast<int64_t>(g) * m3 + h;
            width[g] = std::max<int>(width[g], static_cast<int>(S.rowptr[row + 1] - S.rowptr[row]));
        }
    d.ell_off[0] = 0;
    for (int g = 0; g < 8; ++g) d.ell_off[g + 1] = d.ell_off[g] + width[g] * m3;
    std::vector<int32_t> col(d.ell_off[8], 0);
    std::vector<double> val(2 * static_cast<size_t>(d.ell_off[8]), 0.0);
    for (int g = 0; g < 8; ++g)
        for (int h0 = 0; h0 < m3; h0 += 8) {  // one quarter-warp phase: lanes h0 .. h0+7
            const int lanes = std::min(8, m3 - h0);
            std::vector<std::vector<int64_t>> left(lanes);  // remaining entry indices per lane
            for (int l = 0; l < lanes; ++l) {
                const int64_t row = static_cast<int64_t>(g) * m3 + h0 + l;
                for (int64_t k = S.rowptr[row]; k < S.rowptr[row + 1]; ++k) left[l].push_back(k);
            }
            for (int e = 0; e < width[g]; ++e) {
                unsigned used = 0;
                std::vector<int64_t> pick(lanes, -1);
                for (int l = 0; l < lanes; ++l) {  // distinct bank groups first
                    for (size_t q = 0; q < left[l].size(); ++q)
                        if (!(used & (1u << (S.col[left[l][q]] & 7)))) {
                            pick[l] = left[l][q];
                            left[l].erase(left[l].begin() + static_cast<std::ptrdiff_t>(q));
                            break;
                        }
                    if (pick[l] >= 0) used |= 1u << (S.col[pick[l]] & 7);
                }
                for (int l = 0; l < lanes; ++l) {
                    const int64_t idx = d.ell_off[g] + static_cast<int64_t>(e) * m3 + h0 + l;
                    if (pick[l] < 0 && !left[l].empty()) {  // a conflicting entry is better than a later step
                        pick[l] = left[l].front();
                        left[l].erase(left[l].begin());
                    }
                    if (pick[l] >= 0) {
                        col[idx] = S.col[pick[l]];
                        val[2 * idx] = static_cast<double>(S.val[pick[l]].real());
                        val[2 * idx + 1] = static_cast<double>(S.val[pick[l]].imag());
                    } else {  // padding: any position with a free bank group
                        int b = 0;
                        while (b < 7 && (used & (1u << b))) ++b;
                        used |= 1u << b;
                        col[idx] = b;
                    }
                }
            }
        }
    auto bc = upload(col);
    auto bv = upload(val);
    rt.bufs.insert(rt.bufs.end(), {bc, bv});
    d.col = static_cast<const int*>(bc->ptr);
    d.val = static_cast<const double2*>(bv->ptr);
}

bool tree_matches(const PlanNode& a, const PlanNode& b, long double tol);

void build_two_level(fcct_plan_s* pl) {
    const PlanNode& root = *pl->tree;
    if (root.n != 16) return;
    for (const auto& c : root.children)
        if (!c->radix || c->n != 8) return;
    const int N = static_cast<int>(cube(root.n)), m3 = N / 8;
    const auto perm64 = radix_permutation(root.n);
    std::vector<int32_t> perm(N), pinv(N);
    for (int i = 0; i < N; ++i) {
        perm[i] = static_cast<int32_t>(perm64[i]);
        pinv[perm[i]] = i;
    }
    for (int dir = 0; dir < 2; ++dir) {
        const bool inv = dir == 1;
        RootTables& rt = inv ? pl->rinv : pl->rfwd;
        rt = RootTables{};
        RootDesc& d = rt.desc;
        d.N = N;
        d.m3 = m3;
        d.lgN = 0;
        while ((1 << d.lgN) < N) ++d.lgN;
        build_root_ell(inv ? root.Binv : root.B, N, rt, d);
        std::vector<double> K(128);
        const auto& Kq = inv ? root.Kinv : root.K;
        for (int i = 0; i < 64; ++i) {
            K[2 * i] = static_cast<double>(Kq[i].real());
            K[2 * i + 1] = static_cast<double>(Kq[i].imag());
        }
        auto bk = upload(K), bp = upload(perm), bi = upload(pinv);
        rt.bufs.insert(rt.bufs.end(), {bk, bp, bi});
        d.K = static_cast<const double2*>(bk->ptr);
        d.perm = static_cast<const int*>(bp->ptr);
        d.pinv = static_cast<const int*>(bi->ptr);
    }
    // children: the orbit-FFT executor when every child is the exact n = 8 tree
    // (FCCT_CHILD_PIPELINE=v2 keeps them on the stage pipeline)
    pl->child_offt = pl->exec_force != FCCT_EXEC_TWO_LEVEL_V2;
    for (int c = 0; c < 8 && pl->child_offt; ++c) {
        const PlanNode& ch = *root.children[c];
        OrbitFftHost hf, hi;
        if (!tree_matches(ch, *build_tree(8, ch.p), 1e-9L) || !compile_orbit_fft(8, ch.p, false, hf, kOfBcWarps) ||
            !compile_orbit_fft(8, ch.p, true, hi, kOfBcWarps)) {
            pl->child_offt = false;
            break;
        }
        upload_orbit_fft(hf, pl->ocfwd[c]);
        upload_orbit_fft(hi, pl->ocinv[c]);
        for (auto* t : {&pl->ocfwd[c], &pl->ocinv[c]}) t->desc.in_stride = t->desc.out_stride = 16 * static_cast<int64_t>(N);
    }
    for (int c = 0; c < 8 && !pl->child_offt; ++c) {
        Pipeline2Host hf, hi;
        if (!compile_pipeline2(*root.children[c], false, Shape2{}, hf) ||
            !compile_pipeline2(*root.children[c], true, Shape2{}, hi))
            return;
        upload_pipeline2(hf, pl->cfwd[c]);
        upload_pipeline2(hi, pl->cinv[c]);
        for (auto* t : {&pl->cfwd[c], &pl->cinv[c]}) t->desc.row_in = t->desc.row_out = 2 * static_cast<int64_t>(N);
    }
    pl->two_level = true;
}

// Two-pass orbit-FFT executor: forward S_n (pass A) then F_n (pass B) through a
// complex128 scratch z; inverse F_n^{-1} then S_n^{-1} / n^3.
void run_o16(fcct_plan_s* pl, bool inverse, const void* in, int in_mode, void* out, int out_mode, int64_t batch,
             cudaStream_t st) {
    const size_t bytes = static_cast<size_t>(batch * cube(pl->n) * 16);
    std::lock_guard<std::mutex> lock(pl->scratch_mu);
    if (!pl->scratch0 || pl->scratch0->bytes < bytes) {
        scratch_retire(pl, st);
        pl->scratch0 = std::make_shared<DevBuf>(bytes);
    }
    if (inverse && (!pl->scratch1 || pl->scratch1->bytes < bytes)) {
        scratch_retire(pl, st);
        pl->scratch1 = std::make_shared<DevBuf>(bytes);
    }
    void* z = pl->scratch0->ptr;
    scratch_acquire(pl, st);
    if (!inverse) {
        ck(launch_orbit16_base(pl->o16fwd.desc, in_mode, OF_C128, in, z, batch, st, pl->num_sms), "orbit base change");
        ck(launch_fft_cube(pl->n, +1, OF_C128, out_mode, z, out, batch, pl->o16fwd.desc.zperm, st, pl->num_sms),
           "cube FFT");
    } else {
        ck(launch_fft_cube(pl->n, -1, in_mode, OF_C128, in, z, batch, pl->o16inv.desc.zperm, st, pl->num_sms),
           "cube FFT");
        // rows in orbit order (contiguous stores), then back to natural positions
        ck(launch_orbit16_base(pl->o16inv.desc, OF_C128, out_mode, z, pl->scratch1->ptr, batch, st, pl->num_sms),
           "orbit base change");
        ck(launch_unpermute(out_mode, pl->scratch1->ptr, out, static_cast<int>(cube(pl->n)), batch,
                            pl->o16inv.desc.zperm, st, pl->num_sms),
           "orbit-order rows to natural");
    }
    scratch_release(pl, st);
}

// in_mode / out_mode of the natural side: 0 complex128, 1 complex64, 2 real f64, 3 real f32
void run_two_level(fcct_plan_s* pl, bool inverse, const void* in, int in_mode, void* out, int out_mode, int64_t batch,
                   cudaStream_t st) {
    const int64_t N = cube(pl->n), m3 = N / 8;
    const size_t bytes = static_cast<size_t>(batch * N * 16);
    std::lock_guard<std::mutex> lock(pl->scratch_mu);
    if (!pl->scratch0 || pl->scratch0->bytes < bytes) {
        scratch_retire(pl, st);
        pl->scratch0 = std::make_shared<DevBuf>(bytes);
        pl->scratch1 = std::make_shared<DevBuf>(bytes);
    }
    scratch_acquire(pl, st);
    double* s1 = static_cast<double*>(pl->scratch0->ptr);
    double* s2 = static_cast<double*>(pl->scratch1->ptr);
    for (int k = 0; k < 4; ++k)
        if (!pl->cs[k]) ck(cudaStreamCreateWithFlags(&pl->cs[k], cudaStreamNonBlocking), "stream");
    for (int k = 0; k < 5; ++k)
        if (!pl->cev[k]) ck(cudaEventCreateWithFlags(&pl->cev[k], cudaEventDisableTiming), "event");
    // the eight child pipelines on four streams: one launch's tail overlaps the next one's start
    auto children = [&](Pipeline2Tables* tabs) {
        ck(cudaEventRecord(pl->cev[4], st), "event");
        for (int k = 0; k < 4; ++k) ck(cudaStreamWaitEvent(pl->cs[k], pl->cev[4], 0), "wait");
        const bool inv = tabs == pl->cinv;
        for (int c = 0; c < 8; ++c) {
            if (pl->child_offt)
                ck(launch_orbit_fft(inv ? pl->ocinv[c].desc : pl->ocfwd[c].desc, OF_C128, OF_C128, s1 + 2 * c * m3,
                                    s2 + 2 * c * m3, batch, pl->cs[c & 3], pl->num_sms),
                   "child orbit-FFT");
            else
                ck(launch_pipeline2(tabs[c].desc, s1 + 2 * c * m3, s2 + 2 * c * m3, batch, pl->cs[c & 3], pl->num_sms),
                   "child pipeline");
        }
        for (int k = 0; k < 4; ++k) {
            ck(cudaEventRecord(pl->cev[k], pl->cs[k]), "event");
            ck(cudaStreamWaitEvent(st, pl->cev[k], 0), "wait");
        }
    };
    if (!inverse) {
        ck(launch_root_forward(pl->rfwd.desc, in, in_mode, s1, batch, st, pl->num_sms), "root pass");
        children(pl->cfwd);
        ck(launch_child_to_natural(pl->rfwd.desc, s2, out, out_mode, batch, st), "radix permutation");
    } else {
        ck(launch_natural_to_child(pl->rinv.desc, in, in_mode, s1, batch, st), "radix permutation");
        children(pl->cinv);
        ck(launch_root_inverse(pl->rinv.desc, s2, out, out_mode, batch, st, pl->num_sms), "root pass");
    }
    scratch_release(pl, st);
}

// max |a - b| over the union of the two sparsity patterns
long double sparse_max_diff(const SparseLD& a, const SparseLD& b) {
    if (a.dim != b.dim) return 1e300L;
    long double worst = 0;
    std::vector<cld> row(static_cast<size_t>(a.dim), cld{0, 0});
    for (int64_t r = 0; r < a.dim; ++r) {
        for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) row[a.col[k]] += a.val[k];
        for (int64_t k = b.rowptr[r]; k < b.rowptr[r + 1]; ++k) row[b.col[k]] -= b.val[k];
        for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
            worst = std::max(worst, std::abs(row[a.col[k]]));
            row[a.col[k]] = cld{0, 0};
        }
        for (int64_t k = b.rowptr[r]; k < b.rowptr[r + 1]; ++k) {
            worst = std::max(worst, std::abs(row[b.col[k]]));
            row[b.col[k]] = cld{0, 0};
        }
    }
    return worst;
}

// True when every factor of `a` equals the exact derivation `b` to within
// `tol` (a tree loaded from a plan file, or one built here). A perturbed or
// foreign factor keeps the plan on the stage-by-stage executors, which apply
// the tree's factors as they are (with_perturbed_basis, transform.cpp:542-554).
bool tree_matches(const PlanNode& a, const PlanNode& b, long double tol) {
    if (a.n != b.n || a.radix != b.radix) return false;
    if (!a.radix) {
        if (a.D.size() != b.D.size()) return false;
        for (size_t i = 0; i < a.D.size(); ++i)
            if (std::abs(a.D[i] - b.D[i]) > tol) return false;
        return true;
    }
    for (int i = 0; i < 64; ++i)
        if (std::abs(a.K[i] - b.K[i]) > tol) return false;
    if (sparse_max_diff(a.B, b.B) > tol) return false;
    for (int c = 0; c < 8; ++c)
        if (!tree_matches(*a.children[c], *b.children[c], tol)) return false;
    return true;
}

// The orbit-FFT executors compute F_n S_n(p), i.e. the exact factorisation: a
// tree built here is exact by construction; a loaded (PlanStore) or perturbed
// tree is compared against a fresh derivation.
bool tree_is_exact(const fcct_plan_s* pl) {
    return pl->tree_exact || tree_matches(*pl->tree, *build_tree(pl->n, pl->p), 1e-9L);
}

// Orbit-FFT executor for n = 4, 8: the radix tree telescoped to S_n then the
// radix-2 FFT (orbit_fft.hpp). Valid when the plan's tree is the exact
// factorisation of D_n(p) (it then represents F_n S_n(p) exactly).
void build_orbit_fft(fcct_plan_s* pl) {
    pl->offt = false;
    if (pl->n != 4 && pl->n != 8) return;
    if (!tree_is_exact(pl)) return;
    // default: the warp-specialised kernel (12 base-change + 4 FFT warps);
    // FCCT_EXEC_ORBIT_PHASED selects the phased one (16 warps alternate both roles)
    const int warps = pl->exec_force == FCCT_EXEC_ORBIT_PHASED ? kOfWarps : kOfBcWarps;
    OrbitFftHost hf, hi;
    if (!compile_orbit_fft(pl->n, pl->p, false, hf, warps) || !compile_orbit_fft(pl->n, pl->p, true, hi, warps)) return;
    upload_orbit_fft(hf, pl->ofwd);
    upload_orbit_fft(hi, pl->ofinv);
    pl->offt = true;
}

// Picks the executor of a fast plan: the orbit-FFT executor (n = 4, 8), the
// fp64 DMMA stage pipeline (n <= 8, stage by stage through the tree), the
// two-level executor (n = 16), the shared-memory tile interpreter (one
// block's state fits a CTA tile), else the global-memory multi-pass pipeline.
// fcct_plan_create_executor forces one (fcct_executor: parity tests of every
// executor, A/B runs).
void build_fast_paths(fcct_plan_s* pl) {
    const int x = pl->exec_force;
    const std::string f = x == FCCT_EXEC_AUTO                                   ? ""
                          : x == FCCT_EXEC_ORBIT || x == FCCT_EXEC_ORBIT_PHASED || x == FCCT_EXEC_ORBIT_TWO_PASS ||
                                  x == FCCT_EXEC_ORBIT_STREAMED
                              ? "orbit"
                          : x == FCCT_EXEC_PIPELINE2                           ? "v2"
                          : x == FCCT_EXEC_TWO_LEVEL || x == FCCT_EXEC_TWO_LEVEL_V2 ? "two"
                          : x == FCCT_EXEC_TILE                                ? "v1"
                                                                               : "global";
    const bool f32 = pl->precision == FCCT_F32;
    if (f.empty() || f == "orbit") build_orbit_fft(pl);
    if (pl->offt) return;
    if ((f.empty() || f == "orbit") && x != FCCT_EXEC_ORBIT_TWO_PASS && x != FCCT_EXEC_ORBIT_STREAMED) {  // n = 16: one pass, block resident in shared memory
        pl->opat = false;
        OrbitPatHost hf, hi;
        if (pl->n == 16 && tree_is_exact(pl) && compile_orbit_pat_pair(pl->n, pl->p, hf, hi)) {
            upload_orbit_pat(hf, pl->opfwd);
            upload_orbit_pat(hi, pl->opinv);
            pl->opat = true;
            return;
        }
    }
    if (f.empty() || f == "orbit") {  // n = 16: the two-pass orbit-FFT executor
        pl->o16 = false;
        Orbit16Host hf, hi;
        if (pl->n == 16 && tree_is_exact(pl) &&
            compile_orbit16(pl->n, pl->p, false, hf) && compile_orbit16(pl->n, pl->p, true, hi)) {
            upload_orbit16(hf, pl->o16fwd);
            upload_orbit16(hi, pl->o16inv);
            pl->o16 = true;
            return;
        }
        pl->obig = pl->obpat = false;
        if ((pl->n == 32 || pl->n == 64) && !f32 && x != FCCT_EXEC_ORBIT_STREAMED && tree_is_exact(pl)) {
            OrbitPatHost hf, hi;
            if (compile_orbit_pat_pair(pl->n, pl->p, hf, hi)) {
                upload_orbit_pat_big(hf, pl->obpfwd);
                upload_orbit_pat_big(hi, pl->obpinv);
                pl->obig = pl->obpat = true;
                return;
            }
        }
        if ((pl->n == 32 || pl->n == 64) && !f32 && tree_is_exact(pl)) {
            OrbitBigHost h;
            if (compile_orbit_big(pl->n, pl->p, false, h)) {
                upload_orbit_big(h, pl->obfwd);
                h = OrbitBigHost{};
                if (compile_orbit_big(pl->n, pl->p, true, h)) {
                    upload_orbit_big(h, pl->obinv);
                    pl->obig = true;
                    return;
                }
            }
        }
    }
    if (f.empty() || f == "v2") build_v2(pl);
    if (pl->v2) return;
    if (f.empty() || f == "two") build_two_level(pl);
    if (pl->two_level) return;
    const int tb = choose_tb(cube(pl->n), f32);
    const bool tile_ok = tb > 0 && cube(pl->n) <= 4096;
    if (f == "global" || (f != "v1" && !tile_ok)) {
        if (f32)
            build_global_pipelines<float>(*pl->tree, pl->gfwd, pl->ginv);
        else
            build_global_pipelines<double>(*pl->tree, pl->gfwd, pl->ginv);
        pl->global = true;
        return;
    }
    if (tb == 0) throw FcctError(ST_INVALID_ARGUMENT, "fast pipeline: n too large for one CTA tile");
    if (f32)
        build_pipelines<float>(*pl->tree, tb, pl->fwd, pl->inv);
    else
        build_pipelines<double>(*pl->tree, tb, pl->fwd, pl->inv);
}

void fill_info(fcct_plan_s* pl) {
    fcct_plan_info_t& in = pl->info;
    in.n = pl->n;
    in.r = pl->p.r;
    in.s = pl->p.s;
    in.t = pl->p.t;
    in.kind = pl->radix ? FCCT_KIND_RADIX2 : FCCT_KIND_DIRECT;
    in.method = pl->radix ? FCCT_FAST : FCCT_DIRECT;
    in.precision = pl->precision;
    in.points = cube(pl->n);
    in.executor = !pl->radix ? (pl->tc32 ? 8 : (pl->oz64 ? 9 : 0))
                             : (pl->offt ? 5
                                : (pl->opat ? 10
                                : (pl->o16 ? 6
                                : (pl->obig ? 7 : (pl->v2 ? 2 : (pl->two_level ? 4 : (pl->global ? 3 : 1)))))));
    const double N = static_cast<double>(in.points);
    if (pl->radix) {
        in.levels = tree_levels(pl->n);
        in.tree_nnz = tree_nnz(*pl->tree, false, false);
        in.tree_nnz_inv = tree_nnz(*pl->tree, true, false);
        in.root_nnz = pl->tree->B.nnz();
        in.flops_forward = algorithmic_flops(*pl->tree, false);
        in.flops_inverse = algorithmic_flops(*pl->tree, true);
        in.condition = pl->tree->condition;
        if (pl->offt) {
            in.exec_flops_forward = pl->ofwd.exec_flops;
            in.exec_flops_inverse = pl->ofinv.exec_flops;
        }
        if (pl->o16) {
            in.exec_flops_forward = pl->o16fwd.exec_flops;
            in.exec_flops_inverse = pl->o16inv.exec_flops;
        }
        if (pl->opat) {
            in.exec_flops_forward = pl->opfwd.exec_flops;
            in.exec_flops_inverse = pl->opinv.exec_flops;
            in.exec_flops_forward_real = pl->opfwd.exec_flops_real;
            in.exec_flops_inverse_real = pl->opinv.exec_flops_real;
        }
        if (pl->obig) {
            in.exec_flops_forward = pl->obpat ? pl->obpfwd.exec_flops : pl->obfwd.exec_flops;
            in.exec_flops_inverse = pl->obpat ? pl->obpinv.exec_flops : pl->obinv.exec_flops;
        }
        int64_t bytes = 0;
        for (auto* pt : {&pl->fwd, &pl->inv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->fwd2, &pl->inv2})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->ofwd, &pl->ofinv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->o16fwd, &pl->o16inv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->obfwd, &pl->obinv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->opfwd, &pl->opinv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->obpfwd, &pl->obpinv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->gfwd, &pl->ginv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (auto* pt : {&pl->rfwd, &pl->rinv})
            for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        for (int c = 0; c < 8; ++c) {
            for (auto* pt : {&pl->cfwd[c], &pl->cinv[c]})
                for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
            for (auto* pt : {&pl->ocfwd[c], &pl->ocinv[c]})
                for (auto& b : pt->bufs) bytes += static_cast<int64_t>(b->bytes);
        }
        in.table_bytes = bytes;
        int64_t fwd = 0;
        for (auto* pt : {&pl->obfwd.bufs, &pl->gfwd.bufs, &pl->o16fwd.bufs, &pl->opfwd.bufs, &pl->obpfwd.bufs, &pl->ofwd.bufs, &pl->fwd2.bufs})
            for (auto& b : *pt) fwd += static_cast<int64_t>(b->bytes);
        in.table_bytes_forward = fwd;
    } else {
        in.levels = 0;
        in.flops_forward = in.flops_inverse = 8.0 * N * N;
        // 3xTF32 on tcgen05: three tensor-core products per algorithmic one
        if (pl->tc32) in.exec_flops_forward = in.exec_flops_inverse = 3.0 * 8.0 * N * N;
        // Ozaki: 28 int8 products per algorithmic one (ops, not fp64 flops)
        if (pl->oz64) {
            in.exec_flops_forward = 28.0 * 8.0 * N * N;  // 7 slices: 28 int8 products
            in.exec_flops_inverse = 36.0 * 8.0 * N * N;  // 8 slices: 36
        }
    }
}

// NVTX ranges: plan construction always; the forward / inverse calls in a build with
// FCCT_NVTX=1 (-DFCCT_NVTX: the single-transform latency config is a few microseconds per
// call, so the apply path carries no instrumentation by default).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

fcct_plan_s* create_plan(int n, const Params& p, int method, int precision, int device,
                         PlanStore* store = nullptr, int executor = FCCT_EXEC_AUTO) {
    NvtxRange range(method == FCCT_FAST ? "fcct build_plan" : "fcct dense_transform");
    if (executor < FCCT_EXEC_AUTO || executor > FCCT_EXEC_ORBIT_STREAMED)
        throw FcctError(ST_INVALID_ARGUMENT, "unknown executor");
    if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "build_plan: n must be >= 1");
    if (method != FCCT_DIRECT && method != FCCT_FAST) throw FcctError(ST_INVALID_ARGUMENT, "unknown method");
    if (precision != FCCT_F64 && precision != FCCT_F32) throw FcctError(ST_INVALID_ARGUMENT, "unknown precision");
    if (!std::isfinite(p.r) || !std::isfinite(p.s) || !std::isfinite(p.t))
        throw FcctError(ST_INVALID_ARGUMENT, "grid offsets must be finite");
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw FcctError(ST_INVALID_ARGUMENT, "no such CUDA device");
    DeviceGuard guard(device);
    g_colnorm_device.store(device);
    auto pl = std::make_unique<fcct_plan_s>();
    pl->n = n;
    pl->p = p;
    pl->precision = precision;
    pl->device = device;
    pl->exec_force = executor;
    ck(cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    const bool f32 = precision == FCCT_F32;
    const bool radix = method == FCCT_FAST && n % 2 == 0;
    if (radix) {
        if (store) {
            check_nodes(n, p);
            pl->tree = store->load_or_build(n, p);
        } else {
            pl->tree = build_tree(n, p);  // degeneracy + condition gates inside
            pl->tree_exact = true;
        }
        pl->radix = true;
        build_fast_paths(pl.get());
    } else {
        check_nodes(n, p);
        pl->radix = false;
        build_direct(pl.get());
    }
    pl->method = pl->radix ? FCCT_FAST : FCCT_DIRECT;
    fill_info(pl.get());
    return pl.release();
}

void run(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st);
void run_real(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st);

// Device buffers that are not 16-byte aligned (a caller's sub-range at an odd
// complex64 / real offset) cannot feed the TMA row copies and vector loads of
// the executors: such calls run on aligned staging copies (the result is the
// same; the staging is the caller's cost). Returns true when it handled the call.
bool run_staged_if_unaligned(fcct_plan_s* pl, bool inverse, bool real_io, const void* in, void* out, int64_t batch,
                             cudaStream_t st) {
    if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) return false;
    const int64_t N = cube(pl->n), eb = elem_bytes(pl);
    const int64_t in_eb = (real_io && !inverse) ? eb / 2 : eb, out_eb = (real_io && inverse) ? eb / 2 : eb;
    DevBuf si(static_cast<size_t>(batch * N * in_eb)), so(static_cast<size_t>(batch * N * out_eb));
    ck(cudaMemcpyAsync(si.ptr, in, si.bytes, cudaMemcpyDeviceToDevice, st), "stage input");
    if (real_io)
        run_real(pl, inverse, si.ptr, so.ptr, batch, st);
    else
        run(pl, inverse, si.ptr, so.ptr, batch, st);
    ck(cudaMemcpyAsync(out, so.ptr, so.bytes, cudaMemcpyDeviceToDevice, st), "copy back");
    ck(cudaStreamSynchronize(st), "sync");  // before the staging buffers are freed
    return true;
}

void run(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st) {
    if (batch < 0) throw FcctError(ST_SIZE_MISMATCH, "batch must be >= 0");
    if (batch == 0) return;
    if (!in || !out) throw FcctError(ST_INVALID_ARGUMENT, "null buffer");
#ifdef FCCT_NVTX
    NvtxRange range(inverse ? "fcct inverse" : "fcct forward");
#endif
    DeviceGuard guard(pl->device);
    if (run_staged_if_unaligned(pl, inverse, false, in, out, batch, st)) return;
    const bool f32 = pl->precision == FCCT_F32;
    if (pl->radix) {
        if (pl->two_level) {
            run_two_level(pl, inverse, in, f32 ? 1 : 0, out, f32 ? 1 : 0, batch, st);
            return;
        }
        if (pl->opat) {
            ck(launch_orbit_pat(inverse ? pl->opinv.desc : pl->opfwd.desc, f32 ? OF_C64 : OF_C128,
                                f32 ? OF_C64 : OF_C128, in, out, batch, st, pl->num_sms),
               "orbit-pattern executor");
            return;
        }
        if (pl->o16) {
            run_o16(pl, inverse, in, f32 ? OF_C64 : OF_C128, out, f32 ? OF_C64 : OF_C128, batch, st);
            return;
        }
        if (pl->obig) {  // S pass + three line-FFT passes through a plan-owned scratch
            const size_t bytes = static_cast<size_t>(batch * cube(pl->n) * 16);
            std::lock_guard<std::mutex> lock(pl->scratch_mu);
            if (!pl->scratch0 || pl->scratch0->bytes < bytes) {
                scratch_retire(pl, st);
                pl->scratch0 = std::make_shared<DevBuf>(bytes);
            }
            void* z = pl->scratch0->ptr;
            scratch_acquire(pl, st);
            if (!inverse) {
                ck(pl->obpat ? launch_orbit_pat_big(pl->obpfwd.desc, in, z, batch, st)
                             : launch_orbit_big_s(pl->obfwd.desc, in, z, batch, st),
                   "orbit base change");
                ck(launch_line_fft(pl->n, 2, +1, z, z, batch, st), "line FFT");
                ck(launch_line_fft(pl->n, 1, +1, z, z, batch, st), "line FFT");
                ck(launch_line_fft(pl->n, 0, +1, z, out, batch, st), "line FFT");
            } else {
                ck(launch_line_fft(pl->n, 0, -1, in, z, batch, st), "line FFT");
                ck(launch_line_fft(pl->n, 1, -1, z, z, batch, st), "line FFT");
                ck(launch_line_fft(pl->n, 2, -1, z, z, batch, st), "line FFT");
                ck(pl->obpat ? launch_orbit_pat_big(pl->obpinv.desc, z, out, batch, st)
                             : launch_orbit_big_s(pl->obinv.desc, z, out, batch, st),
                   "orbit base change");
            }
            scratch_release(pl, st);
            return;
        }
        if (pl->offt) {
            const int m = f32 ? OF_C64 : OF_C128;
            ck(launch_orbit_fft(inverse ? pl->ofinv.desc : pl->ofwd.desc, m, m, in, out, batch, st, pl->num_sms),
               "orbit-FFT executor");
            return;
        }
        if (pl->v2) {
            ck(launch_pipeline2(inverse ? pl->inv2.desc : pl->fwd2.desc, in, out, batch, st, pl->num_sms),
               "fast pipeline v2");
        } else if (pl->global) {
            const size_t bytes = static_cast<size_t>(batch * cube(pl->n) * elem_bytes(pl));
            std::lock_guard<std::mutex> lock(pl->scratch_mu);
            if (!pl->scratch0 || pl->scratch0->bytes < bytes) {
                scratch_retire(pl, st);
                pl->scratch0 = std::make_shared<DevBuf>(bytes);
                pl->scratch1 = std::make_shared<DevBuf>(bytes);
            }
            scratch_acquire(pl, st);
            ck(launch_global_pipeline(inverse ? pl->ginv.desc : pl->gfwd.desc, f32, in, out, pl->scratch0->ptr,
                                      pl->scratch1->ptr, batch, st),
               "global pipeline");
            scratch_release(pl, st);
        } else
            ck(launch_pipeline(inverse ? pl->inv.desc : pl->fwd.desc, f32, in, out, batch, st, pl->num_sms),
               "fast pipeline");
        return;
    }
    const int64_t N = cube(pl->n);
    const void* W = inverse ? pl->Wt_inv->ptr : pl->Wt_fwd->ptr;
    void* dst = out;
    std::shared_ptr<DevBuf> tmp, tmp_in;
    const size_t io_bytes = static_cast<size_t>(batch * N * elem_bytes(pl));
    // the tcgen05 paths read rows with TMA / 32-byte vector loads: buffers that are
    // not 32-byte aligned (a caller's sub-range at an odd offset) are staged
    const bool misaligned = (pl->oz64 || pl->tc32) &&
                            ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 31) != 0;
    if (misaligned && (reinterpret_cast<uintptr_t>(in) & 31) != 0) {
        tmp_in = std::make_shared<DevBuf>(io_bytes);
        ck(cudaMemcpyAsync(tmp_in->ptr, in, io_bytes, cudaMemcpyDeviceToDevice, st), "stage input");
        in = tmp_in->ptr;
    }
    if (in == out || (misaligned && (reinterpret_cast<uintptr_t>(out) & 31) != 0)) {
        tmp = std::make_shared<DevBuf>(io_bytes);
        dst = tmp->ptr;
    }
    if (pl->oz64) {
        const int K = static_cast<int>(2 * N);
        // the slice workspace is plan-owned scratch: ordered across streams by the
        // plan's scratch event like the other executors' scratch
        std::lock_guard<std::mutex> lock(pl->scratch_mu);
        const size_t need = static_cast<size_t>(ozaki_slices()) * batch * K;
        if (!pl->oz_in || pl->oz_in->bytes < need || pl->oz_in_scale->bytes < static_cast<size_t>(batch) * 8) {
            scratch_retire(pl, st);
            pl->oz_in = std::make_shared<DevBuf>(need);
            pl->oz_in_scale = std::make_shared<DevBuf>(static_cast<size_t>(batch) * 8);
        }
        scratch_acquire(pl, st);
        const int S = inverse ? kOzaki_inverse : kOzaki_forward;
        ck(ozaki_slice(static_cast<const double*>(in), batch, K, S, static_cast<int8_t*>(pl->oz_in->ptr),
                       static_cast<double*>(pl->oz_in_scale->ptr), st),
           "ozaki input slices");
        ck(launch_gemm_ozaki(static_cast<const int8_t*>(pl->oz_in->ptr), static_cast<const double*>(pl->oz_in_scale->ptr),
                             static_cast<const int8_t*>(pl->oz_w[inverse ? 1 : 0]->ptr),
                             static_cast<const double*>(pl->oz_ws[inverse ? 1 : 0]->ptr), static_cast<double*>(dst),
                             batch, K, K, S, pl->num_sms, st),
           "direct gemm ozaki (tcgen05 int8)");
        scratch_release(pl, st);
    } else if (pl->tc32)
        ck(launch_gemm_tf32x3(static_cast<const float*>(in), static_cast<const float*>(W),
                              static_cast<const float*>(inverse ? pl->Wt_inv_lo->ptr : pl->Wt_fwd_lo->ptr),
                              static_cast<float*>(dst), batch, static_cast<int>(2 * N), static_cast<int>(2 * N),
                              pl->num_sms, st),
           "direct gemm tf32x3 (tcgen05)");
    else if (f32)
        ck(launch_gemm_f32(static_cast<const float*>(in), static_cast<const float*>(W), static_cast<float*>(dst),
                           batch, static_cast<int>(2 * N), static_cast<int>(2 * N), st),
           "direct gemm f32");
    else
        ck(launch_gemm_f64(static_cast<const double*>(in), static_cast<const double*>(W), static_cast<double*>(dst),
                           batch, static_cast<int>(2 * N), static_cast<int>(2 * N), st),
           "direct gemm f64");
    if (tmp)
        ck(cudaMemcpyAsync(out, tmp->ptr, static_cast<size_t>(batch * N * elem_bytes(pl)), cudaMemcpyDeviceToDevice, st),
           "copy back");
    if (tmp || tmp_in) ck(cudaStreamSynchronize(st), "sync");  // before the staging buffers are freed
}

void run(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st);
void run_real(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st);

// Host-buffer calls: the batch is cut into chunks that alternate between two
// streams, so the H2D copy of one chunk, the transform of the previous one
// and the D2H copy of the one before overlap (both copy directions run at
// once over PCIe / C2C; pinned host buffers give fully asynchronous DMA).
void run_host_any(fcct_plan_s* pl, bool inverse, bool real_io, const void* in, void* out, int64_t batch,
                  cudaStream_t st) {
    if (batch < 0) throw FcctError(ST_SIZE_MISMATCH, "batch must be >= 0");
    if (batch == 0) return;
    if (!in || !out) throw FcctError(ST_INVALID_ARGUMENT, "null buffer");
    DeviceGuard guard(pl->device);
    const int64_t N = cube(pl->n), eb = elem_bytes(pl);
    const int64_t in_eb = (real_io && !inverse) ? eb / 2 : eb, out_eb = (real_io && inverse) ? eb / 2 : eb;
    const int64_t block_bytes = N * eb;
    // ~32 MB chunks (at least 8 per call when the batch is large), whole blocks
    // chunk size: FCCT_HOST_CHUNK_MB (default 32 MB), at least 8 chunks per call
    int64_t chunk_mb = 32;
    if (const char* e = ab_env("FCCT_HOST_CHUNK_MB")) chunk_mb = std::max<int64_t>(1, std::atoll(e));
    int64_t chunk = std::max<int64_t>(1, (chunk_mb << 20) / block_bytes);
    chunk = std::min(chunk, std::max<int64_t>(1, (batch + 7) / 8));
    chunk = std::min(chunk, batch);
    const size_t ws_bytes = static_cast<size_t>(chunk * block_bytes);
    std::lock_guard<std::mutex> lock(pl->ws_mu);
    for (int k = 0; k < 2; ++k) {
        if (!pl->hs[k]) ck(cudaStreamCreateWithFlags(&pl->hs[k], cudaStreamNonBlocking), "stream");
        if (!pl->ws_in[k] || pl->ws_in[k]->bytes < ws_bytes) {
            pl->ws_in[k] = std::make_shared<DevBuf>(ws_bytes);
            pl->ws_out[k] = std::make_shared<DevBuf>(ws_bytes);
        }
    }
    if (!pl->hev) ck(cudaEventCreateWithFlags(&pl->hev, cudaEventDisableTiming), "event");
    // work already queued on the caller's stream comes first
    ck(cudaEventRecord(pl->hev, st), "event record");
    for (auto h : pl->hs) ck(cudaStreamWaitEvent(h, pl->hev, 0), "stream wait");
    const char* src = static_cast<const char*>(in);
    char* dst = static_cast<char*>(out);
    // Pageable caller memory (e.g. a std::vector / Eigen::VectorXcd) is staged
    // through pinned bounce buffers: the host copy into slot c & 1 overlaps the
    // device work of chunk c - 1, and the copy out of chunk c - 1 overlaps
    // chunk c. Pinned caller memory is DMA'd directly.
    const bool stage_in = is_pageable_host(in), stage_out = is_pageable_host(out);
    if (stage_in || stage_out) {
        for (int k = 0; k < 2; ++k) {
            if (stage_in) pl->pin_in[k].reserve(static_cast<size_t>(chunk * N * in_eb));
            if (stage_out) pl->pin_out[k].reserve(static_cast<size_t>(chunk * N * out_eb));
            if (!pl->h2d_ev[k]) ck(cudaEventCreateWithFlags(&pl->h2d_ev[k], cudaEventDisableTiming), "event");
            if (!pl->d2h_ev[k]) ck(cudaEventCreateWithFlags(&pl->d2h_ev[k], cudaEventDisableTiming), "event");
        }
    }
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    auto copy_out = [&](int64_t c) {  // host side of chunk c's D2H (staged output only)
        const int64_t off = c * chunk, nb = std::min(chunk, batch - off);
        ck(cudaEventSynchronize(pl->d2h_ev[c & 1]), "D2H wait");
        par_memcpy(dst + off * N * out_eb, pl->pin_out[c & 1].ptr, static_cast<size_t>(nb * N * out_eb));
    };
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t off = c * chunk, nb = std::min(chunk, batch - off);
        const int k = static_cast<int>(c & 1);
        cudaStream_t h = pl->hs[k];
        void* wi = pl->ws_in[k]->ptr;
        void* wo = pl->ws_out[k]->ptr;
        const size_t ib = static_cast<size_t>(nb * N * in_eb), ob = static_cast<size_t>(nb * N * out_eb);
        const void* hsrc = src + off * N * in_eb;
        if (stage_in) {
            if (c >= 2) ck(cudaEventSynchronize(pl->h2d_ev[k]), "H2D wait");  // chunk c - 2 has left the slot
            par_memcpy(pl->pin_in[k].ptr, hsrc, ib);
            hsrc = pl->pin_in[k].ptr;
        }
        ck(cudaMemcpyAsync(wi, hsrc, ib, cudaMemcpyHostToDevice, h), "H2D");
        if (stage_in) ck(cudaEventRecord(pl->h2d_ev[k], h), "event record");
        if (real_io)
            run_real(pl, inverse, wi, wo, nb, h);
        else
            run(pl, inverse, wi, wo, nb, h);
        ck(cudaMemcpyAsync(stage_out ? pl->pin_out[k].ptr : static_cast<void*>(dst + off * N * out_eb), wo, ob,
                           cudaMemcpyDeviceToHost, h),
           "D2H");
        if (stage_out) {
            ck(cudaEventRecord(pl->d2h_ev[k], h), "event record");
            if (c >= 1) copy_out(c - 1);  // slot (c - 1) & 1 is reused by chunk c + 1
        }
    }
    if (stage_out) copy_out(nchunks - 1);
    for (auto h : pl->hs) ck(cudaStreamSynchronize(h), "sync");
}

void run_host(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st) {
    run_host_any(pl, inverse, false, in, out, batch, st);
}

// Real-sample I/O: forward takes real samples (z_transform, voxel_io.cpp:178-186),
// inverse returns real parts (grid_from_signal, voxel_io.cpp:188-198). The v2
// pipeline fuses both into its tile load / store; the other executors stage
// through a complex workspace.
void run_real(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st) {
    if (batch < 0) throw FcctError(ST_SIZE_MISMATCH, "batch must be >= 0");
    if (batch == 0) return;
    if (!in || !out) throw FcctError(ST_INVALID_ARGUMENT, "null buffer");
#ifdef FCCT_NVTX
    NvtxRange range(inverse ? "fcct inverse (real output)" : "fcct forward (real input)");
#endif
    DeviceGuard guard(pl->device);
    if (run_staged_if_unaligned(pl, inverse, true, in, out, batch, st)) return;
    const bool f32 = pl->precision == FCCT_F32;
    if (pl->radix && pl->two_level) {
        const int cm = f32 ? 1 : 0, rm = f32 ? 3 : 2;
        run_two_level(pl, inverse, in, inverse ? cm : rm, out, inverse ? rm : cm, batch, st);
        return;
    }
    if (pl->radix && pl->opat) {
        const int cm = f32 ? OF_C64 : OF_C128, rm = f32 ? OF_R32 : OF_R64;
        ck(launch_orbit_pat(inverse ? pl->opinv.desc : pl->opfwd.desc, inverse ? cm : rm, inverse ? rm : cm, in, out,
                            batch, st, pl->num_sms),
           "orbit-pattern executor (real I/O)");
        return;
    }
    if (pl->radix && pl->o16) {
        const int cm = f32 ? OF_C64 : OF_C128, rm = f32 ? OF_R32 : OF_R64;
        run_o16(pl, inverse, in, inverse ? cm : rm, out, inverse ? rm : cm, batch, st);
        return;
    }
    if (pl->radix && pl->offt) {
        const int cm = f32 ? OF_C64 : OF_C128, rm = f32 ? OF_R32 : OF_R64;
        ck(launch_orbit_fft(inverse ? pl->ofinv.desc : pl->ofwd.desc, inverse ? cm : rm, inverse ? rm : cm, in, out,
                            batch, st, pl->num_sms),
           "orbit-FFT executor (real I/O)");
        return;
    }
    if (pl->radix && pl->v2) {
        Pipeline2Desc d = inverse ? pl->inv2.desc : pl->fwd2.desc;
        (inverse ? d.real_out : d.real_in) = 1;
        ck(launch_pipeline2(d, in, out, batch, st, pl->num_sms), "fast pipeline v2 (real I/O)");
        return;
    }
    const int64_t count = batch * cube(pl->n);
    const size_t bytes = static_cast<size_t>(count * elem_bytes(pl));
    std::lock_guard<std::mutex> lock(pl->ws_real_mu);
    if (!pl->ws_real || pl->ws_real->bytes < bytes) {
        ck(cudaStreamSynchronize(st), "sync");
        pl->ws_real = std::make_shared<DevBuf>(bytes);
    }
    if (inverse) {
        run(pl, true, in, pl->ws_real->ptr, batch, st);
        ck(launch_real_part(pl->ws_real->ptr, out, count, f32, st), "real part");
    } else {
        ck(launch_complexify(in, pl->ws_real->ptr, count, f32, st), "complexify");
        run(pl, false, pl->ws_real->ptr, out, batch, st);
    }
    ck(cudaStreamSynchronize(st), "sync");  // the plan-owned workspace serialises calls on this path
}

void run_real_host(fcct_plan_s* pl, bool inverse, const void* in, void* out, int64_t batch, cudaStream_t st) {
    run_host_any(pl, inverse, true, in, out, batch, st);
}

template <typename F>
fcct_status guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return FCCT_OK;
    } catch (const FcctError& e) {
        g_last_error = e.what();
        return static_cast<fcct_status>(e.code);
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FCCT_INVALID_ARGUMENT;
    }
}

}  // namespace

extern "C" {

const char* fcct_last_error(void) { return g_last_error.c_str(); }

fcct_status fcct_plan_create(int n, double r, double s, double t, int method, int precision, int device,
                             fcct_plan* out) {
    return guarded([&] {
        if (!out) throw FcctError(ST_INVALID_ARGUMENT, "null plan pointer");
        *out = create_plan(n, Params{r, s, t}, method, precision, device);
    });
}

fcct_status fcct_plan_create_executor(int n, double r, double s, double t, int precision, int device, int executor,
                                      fcct_plan* out) {
    return guarded([&] {
        if (!out) throw FcctError(ST_INVALID_ARGUMENT, "null plan pointer");
        *out = create_plan(n, Params{r, s, t}, FCCT_FAST, precision, device, nullptr, executor);
    });
}

fcct_status fcct_plan_destroy(fcct_plan plan) {
    return guarded([&] {
        if (!plan) return;
        DeviceGuard guard(plan->device);
        cudaDeviceSynchronize();
        delete plan;
    });
}

fcct_status fcct_plan_info(fcct_plan plan, fcct_plan_info_t* info) {
    return guarded([&] {
        if (!plan || !info) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        *info = plan->info;
    });
}

fcct_status fcct_forward(fcct_plan plan, const void* in, void* out, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run(plan, false, in, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_inverse(fcct_plan plan, const void* in, void* out, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run(plan, true, in, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_inverse_checked(fcct_plan plan, double r, double s, double t, const void* in, void* out,
                                 int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        if (!(Params{r, s, t} == plan->p))
            throw FcctError(ST_PARAMS_MISMATCH, "inverse_apply: spectrum was produced on a different skew grid");
        run(plan, true, in, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_forward_host(fcct_plan plan, const void* in, void* out, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run_host(plan, false, in, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_inverse_host(fcct_plan plan, const void* in, void* out, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run_host(plan, true, in, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_forward_real(fcct_plan plan, const void* in_real, void* out, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run_real(plan, false, in_real, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_inverse_real(fcct_plan plan, const void* in, void* out_real, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run_real(plan, true, in, out_real, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_forward_real_host(fcct_plan plan, const void* in_real, void* out, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run_real_host(plan, false, in_real, out, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_inverse_real_host(fcct_plan plan, const void* in, void* out_real, int64_t batch, void* stream) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        run_real_host(plan, true, in, out_real, batch, static_cast<cudaStream_t>(stream));
    });
}

fcct_status fcct_radix_permutation(int n, uint64_t* out_host) {
    return guarded([&] {
        if (n < 2) throw FcctError(ST_INVALID_ARGUMENT, "radix_permutation: n must be >= 2");
        if (n % 2 != 0) throw FcctError(ST_ODD_SIZE, "radix_permutation: size " + std::to_string(n) + " is odd");
        if (!out_host) throw FcctError(ST_INVALID_ARGUMENT, "null output");
        const int64_t N = cube(n);
        DevBuf d(static_cast<size_t>(N) * 8);
        ck(gen_radix_permutation(n, static_cast<unsigned long long*>(d.ptr), nullptr), "radix permutation");
        ck(cudaMemcpy(out_host, d.ptr, static_cast<size_t>(N) * 8, cudaMemcpyDeviceToHost), "D2H");
    });
}

fcct_status fcct_dense_matrix(int n, double r, double s, double t, void* out_device, void* stream) {
    return guarded([&] {
        if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "dense_transform: n must be >= 1");
        if (!out_device) throw FcctError(ST_INVALID_ARGUMENT, "null output");
        check_nodes(n, Params{r, s, t});  // transform.cpp:132
        ck(gen_dense_colmajor(n, r, s, t, static_cast<double*>(out_device), static_cast<cudaStream_t>(stream)),
           "dense matrix");
    });
}

fcct_status fcct_dense_matrix_host(int n, double r, double s, double t, int device, void* out_host) {
    return guarded([&] {
        if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "dense_transform: n must be >= 1");
        if (!out_host) throw FcctError(ST_INVALID_ARGUMENT, "null output");
        DeviceGuard guard(device);
        check_nodes(n, Params{r, s, t});  // transform.cpp:132
        const size_t bytes = static_cast<size_t>(cube(n)) * cube(n) * 16;
        DevBuf d(bytes);
        ck(gen_dense_colmajor(n, r, s, t, static_cast<double*>(d.ptr), nullptr), "dense matrix");
        ck(cudaMemcpy(out_host, d.ptr, bytes, cudaMemcpyDeviceToHost), "D2H");
    });
}

fcct_status fcct_skew_nodes(int n, double r, double s, double t, void* out_device, void* stream) {
    return guarded([&] {
        if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "skew_nodes: n must be >= 1");
        if (!out_device) throw FcctError(ST_INVALID_ARGUMENT, "null output");
        DevBuf flag(sizeof(int));
        ck(cudaMemset(flag.ptr, 0, sizeof(int)), "memset");
        auto st = static_cast<cudaStream_t>(stream);
        ck(gen_nodes(n, r, s, t, static_cast<double*>(out_device), static_cast<int*>(flag.ptr), st), "nodes");
        int h = 0;
        ck(cudaMemcpyAsync(&h, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        if (h) throw FcctError(ST_DEGENERATE_NODES, "two nodes map to the same spectral point for n=" + std::to_string(n));
    });
}

fcct_status fcct_plan_kernel(fcct_plan plan, double* out128) {
    return guarded([&] {
        if (!plan || !out128) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        if (!plan->radix) throw FcctError(ST_INVALID_ARGUMENT, "kernel(): plan is direct");
        for (int blk = 0; blk < 8; ++blk)
            for (int g = 0; g < 8; ++g) {
                const cld v = plan->tree->K[blk * 8 + g];
                out128[2 * (g * 8 + blk)] = static_cast<double>(v.real());
                out128[2 * (g * 8 + blk) + 1] = static_cast<double>(v.imag());
            }
    });
}

fcct_status fcct_plan_basis(fcct_plan plan, int64_t* nnz, int64_t* colptr, int32_t* rowidx, double* values) {
    return guarded([&] {
        if (!plan || !nnz) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        if (!plan->radix) throw FcctError(ST_INVALID_ARGUMENT, "basis(): plan is direct");
        const SparseLD& B = plan->tree->B;
        *nnz = B.nnz();
        if (!colptr || !rowidx || !values) return;
        // CSR -> CSC (Eigen's compressed column storage, rows sorted per column)
        const int64_t N = B.dim;
        std::vector<int64_t> cnt(N + 1, 0);
        for (int32_t c : B.col) cnt[c + 1]++;
        for (int64_t c = 0; c < N; ++c) cnt[c + 1] += cnt[c];
        std::copy(cnt.begin(), cnt.end(), colptr);
        std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t r = 0; r < N; ++r)
            for (int64_t k = B.rowptr[r]; k < B.rowptr[r + 1]; ++k) {
                const int64_t dst = fill[B.col[k]]++;
                rowidx[dst] = static_cast<int32_t>(r);
                values[2 * dst] = static_cast<double>(B.val[k].real());
                values[2 * dst + 1] = static_cast<double>(B.val[k].imag());
            }
    });
}

fcct_status fcct_plan_child(fcct_plan plan, int index, int* n, double* r, double* s, double* t, int* kind) {
    return guarded([&] {
        if (!plan) throw FcctError(ST_INVALID_ARGUMENT, "null plan");
        if (!plan->radix) throw FcctError(ST_INVALID_ARGUMENT, "children(): plan is direct");
        if (index < 0 || index >= 8) throw FcctError(ST_INVALID_ARGUMENT, "child index out of range");
        const PlanNode& c = *plan->tree->children[index];
        if (n) *n = c.n;
        if (r) *r = c.p.r;
        if (s) *s = c.p.s;
        if (t) *t = c.p.t;
        if (kind) *kind = c.radix ? FCCT_KIND_RADIX2 : FCCT_KIND_DIRECT;
    });
}

fcct_status fcct_factorization_residual(fcct_plan plan, double* out) {
    return guarded([&] {
        if (!plan || !out) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        if (plan->precision != FCCT_F64) throw FcctError(ST_INVALID_ARGUMENT, "residual needs an fp64 plan");
        DeviceGuard guard(plan->device);
        const int64_t N = cube(plan->n);
        DevBuf E(static_cast<size_t>(N * N) * 16), Y(static_cast<size_t>(N * N) * 16), D(static_cast<size_t>(N * N) * 16);
        ck(gen_identity(static_cast<int>(N), E.ptr, false, nullptr), "identity");
        run(plan, false, E.ptr, Y.ptr, N, nullptr);
        ck(gen_dense_colmajor(plan->n, plan->p.r, plan->p.s, plan->p.t, static_cast<double*>(D.ptr), nullptr), "dense");
        const int nb = 512;
        DevBuf part(nb * sizeof(double));
        ck(residual_max(static_cast<const double*>(Y.ptr), static_cast<const double*>(D.ptr), static_cast<int>(N),
                        static_cast<double*>(part.ptr), nb, nullptr),
           "residual");
        std::vector<double> h(nb);
        ck(cudaMemcpy(h.data(), part.ptr, nb * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        *out = *std::max_element(h.begin(), h.end());
    });
}

fcct_status fcct_plan_perturbed_basis(fcct_plan plan, double delta, fcct_plan* out) {
    return guarded([&] {
        if (!plan || !out) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        if (!plan->radix) throw FcctError(ST_INVALID_ARGUMENT, "with_perturbed_basis: plan has no basis factor");
        if (plan->tree->B.nnz() == 0) throw FcctError(ST_INVALID_ARGUMENT, "with_perturbed_basis: basis is empty");
        DeviceGuard guard(plan->device);
        auto root = std::make_shared<PlanNode>(*plan->tree);  // children shared
        // valuePtr()[0] of the CSC basis: column 0, smallest row (transform.cpp:550)
        int64_t best = -1;
        int32_t best_row = INT32_MAX;
        for (int64_t r = 0; r < root->B.dim && best < 0; ++r)
            for (int64_t k = root->B.rowptr[r]; k < root->B.rowptr[r + 1]; ++k)
                if (root->B.col[k] == 0 && r < best_row) {
                    best = k;
                    best_row = static_cast<int32_t>(r);
                    break;
                }
        if (best < 0) throw FcctError(ST_INVALID_ARGUMENT, "with_perturbed_basis: column 0 is empty");
        root->B.val[best] += static_cast<long double>(delta);
        root->Binv = invert_sparse(root->B);  // the reference refactors the perturbed basis (transform.cpp:551-553)
        auto pl = std::make_unique<fcct_plan_s>();
        pl->n = plan->n;
        pl->p = plan->p;
        pl->precision = plan->precision;
        pl->device = plan->device;
        pl->num_sms = plan->num_sms;
        pl->radix = true;
        pl->tree = root;
        build_fast_paths(pl.get());
        pl->method = FCCT_FAST;
        fill_info(pl.get());
        *out = pl.release();
    });
}

struct fcct_store_s {
    std::unique_ptr<PlanStore> store;
};

fcct_status fcct_store_open(const char* dir, fcct_store* out) {
    return guarded([&] {
        if (!dir || !out) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        auto st = std::make_unique<fcct_store_s>();
        st->store = std::make_unique<PlanStore>(dir);
        *out = st.release();
    });
}

fcct_status fcct_store_close(fcct_store store) {
    return guarded([&] { delete store; });
}

fcct_status fcct_store_warm(fcct_store store, int n, double r, double s, double t) {
    return guarded([&] {
        if (!store) throw FcctError(ST_INVALID_ARGUMENT, "null store");
        if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "build_plan: n must be >= 1");
        check_nodes(n, Params{r, s, t});
        (void)store->store->load_or_build(n, Params{r, s, t});
    });
}

fcct_status fcct_store_stats(fcct_store store, int* hits, int* misses, int* rebuilt) {
    return guarded([&] {
        if (!store) throw FcctError(ST_INVALID_ARGUMENT, "null store");
        const auto st = store->store->stats();
        if (hits) *hits = st.hits;
        if (misses) *misses = st.misses;
        if (rebuilt) *rebuilt = st.rebuilt;
    });
}

fcct_status fcct_store_path(fcct_store store, int n, double r, double s, double t, char* buf, int len) {
    return guarded([&] {
        if (!store || !buf || len <= 0) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        const std::string p = store->store->path_for(n, Params{r, s, t});
        if (static_cast<int>(p.size()) >= len) throw FcctError(ST_INVALID_ARGUMENT, "buffer too small");
        std::memcpy(buf, p.c_str(), p.size() + 1);
    });
}

fcct_status fcct_plan_create_from_store(fcct_store store, int n, double r, double s, double t, int precision,
                                        int device, fcct_plan* out) {
    return guarded([&] {
        if (!store || !out) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        *out = create_plan(n, Params{r, s, t}, FCCT_FAST, precision, device, store->store.get());
    });
}

fcct_status fcct_shard_range(int64_t total, int rank, int world, int64_t* begin, int64_t* end) {
    return guarded([&] {
        if (total < 0 || world < 1 || rank < 0 || rank >= world || !begin || !end)
            throw FcctError(ST_INVALID_ARGUMENT, "bad shard arguments");
        const int64_t per = (total + world - 1) / world;
        *begin = std::min<int64_t>(total, per * rank);
        *end = std::min<int64_t>(total, per * (rank + 1));
    });
}

fcct_status fcct_condition_estimate(int n, double r, double s, double t, double* out) {
    return guarded([&] {
        if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "dense_transform: n must be >= 1");
        if (!out) throw FcctError(ST_INVALID_ARGUMENT, "null output");
        const Params p{r, s, t};
        check_nodes(n, p);  // dense_transform runs the degeneracy check (transform.cpp:132)
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) g_colnorm_device.store(dev);
        cudaGetLastError();
        *out = reference_condition(n, p);
    });
}

fcct_status fcct_basis_change(int n, double r, double s, double t, int inverse, int64_t* nnz, int64_t* colptr,
                              int32_t* rowidx, double* values) {
    return guarded([&] {
        if (!nnz) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        if (n < 2 || n % 2 != 0)
            throw FcctError(ST_ODD_SIZE, "basis_change: needs an even size, got " + std::to_string(n));
        static std::mutex mu;
        static std::shared_ptr<const PlanNode> cached;
        std::shared_ptr<const PlanNode> root;
        {
            std::lock_guard<std::mutex> lock(mu);
            if (cached && cached->n == n && cached->p == Params{r, s, t}) root = cached;
        }
        if (!root) {
            root = build_tree(n, Params{r, s, t});
            std::lock_guard<std::mutex> lock(mu);
            cached = root;
        }
        const SparseLD& B = inverse ? root->Binv : root->B;
        *nnz = B.nnz();
        if (!colptr || !rowidx || !values) return;
        const int64_t N = B.dim;
        std::vector<int64_t> cnt(N + 1, 0);
        for (int32_t c : B.col) cnt[c + 1]++;
        for (int64_t c = 0; c < N; ++c) cnt[c + 1] += cnt[c];
        std::copy(cnt.begin(), cnt.end(), colptr);
        std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t row = 0; row < N; ++row)
            for (int64_t k = B.rowptr[row]; k < B.rowptr[row + 1]; ++k) {
                const int64_t dst = fill[B.col[k]]++;
                rowidx[dst] = static_cast<int32_t>(row);
                values[2 * dst] = static_cast<double>(B.val[k].real());
                values[2 * dst + 1] = static_cast<double>(B.val[k].imag());
            }
    });
}

fcct_status fcct_plan_tree_stats(int n, double r, double s, double t, int64_t* tree_nnz_fwd, int64_t* tree_nnz_inv,
                                 double* flops_fwd, double* flops_inv) {
    return guarded([&] {
        if (n < 2 || n % 2 != 0) throw FcctError(ST_ODD_SIZE, "tree stats: needs an even size");
        auto root = build_tree(n, Params{r, s, t});
        if (tree_nnz_fwd) *tree_nnz_fwd = tree_nnz(*root, false, false);
        if (tree_nnz_inv) *tree_nnz_inv = tree_nnz(*root, true, false);
        if (flops_fwd) *flops_fwd = algorithmic_flops(*root, false);
        if (flops_inv) *flops_inv = algorithmic_flops(*root, true);
    });
}

// Host emulation of the v2 DMMA pipeline tables (no GPU): applies the
// compiled stages to `batch` blocks exactly as the kernel indexes them
// (slots, lane-ordered fragments, unit lists). Tests the plan compiler on CPU.
// Host emulation of the large-n orbit-FFT executor's tables (n = 32, 64, CPU tests).
fcct_status fcct_debug_emulate_orbit_big(int n, double r, double s, double t, int inverse, const double* in,
                                         double* out, int64_t batch) {
    return guarded([&] {
        OrbitBigHost h;
        if (!compile_orbit_big(n, Params{r, s, t}, inverse != 0, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by the large-n orbit-FFT executor");
        emulate_orbit_big(h, in, out, batch);
    });
}

// Host emulation of the single-pass orbit-pattern executor's tables (n = 16, CPU
// tests); stats (optional, 6 values): shapes, class sizes, DMMA count, modelled
// shared-memory wavefronts of the gathers / scatters and their floor.
fcct_status fcct_debug_emulate_orbit_pat(int n, double r, double s, double t, int inverse, const double* in,
                                         double* out, int64_t batch, int64_t* stats) {
    return guarded([&] {
        OrbitPatHost h;
        if (!compile_orbit_pat(n, Params{r, s, t}, inverse != 0, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by the orbit-pattern executor");
        if (stats) {
            stats[0] = h.patterns;
            stats[1] = h.cnt[0];
            stats[2] = h.cnt[1];
            stats[3] = h.dmma;
            stats[4] = h.wavefronts;
            stats[5] = h.wavefronts_floor;
        }
        if (batch > 0) emulate_orbit_pat(h, in, out, batch);
    });
}

// Host emulation of the two-pass orbit-FFT executor's tables (n = 16, CPU tests).
fcct_status fcct_debug_emulate_orbit16(int n, double r, double s, double t, int inverse, const double* in, double* out,
                                       int64_t batch) {
    return guarded([&] {
        Orbit16Host h;
        if (!compile_orbit16(n, Params{r, s, t}, inverse != 0, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by the two-pass orbit-FFT executor");
        emulate_orbit16(h, in, out, batch);
    });
}

// Host emulation of the orbit-FFT executor's compiled tables (CPU tests).
fcct_status fcct_debug_emulate_orbit_fft(int n, double r, double s, double t, int inverse, const double* in,
                                         double* out, int64_t batch) {
    return guarded([&] {
        OrbitFftHost h;
        if (!compile_orbit_fft(n, Params{r, s, t}, inverse != 0, h, kOfBcWarps))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by the orbit-FFT executor");
        emulate_orbit_fft(h, in, out, batch);
    });
}

fcct_status fcct_debug_emulate_v2(int n, double r, double s, double t, int inverse, const double* in, double* out,
                                  int64_t batch) {
    return guarded([&] {
        auto root = build_tree(n, Params{r, s, t});
        Pipeline2Host h;
        if (!compile_pipeline2(*root, inverse != 0, Shape2{}, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by pipeline v2");
        const int N = h.N;
        const int kWarps2 = h.shape.warps, kUnits2 = h.shape.units;
        std::vector<double> X(static_cast<size_t>(2) * N), Y(static_cast<size_t>(2) * N);
        for (int64_t b = 0; b < batch; ++b) {
            std::copy(in + 2 * N * b, in + 2 * N * (b + 1), X.begin());
            for (const auto& st : h.stages) {
                std::fill(Y.begin(), Y.end(), 0.0);
                for (int w = 0; w < kWarps2; ++w)
                    for (int j = 0; j < kUnits2; ++j) {
                        const int u = st.warp_units[w * kUnits2 + j];
                        if (u < 0) continue;
                        double acc[8][2] = {};  // [n][part]
                        auto apply = [&](const int slot[4], const double frag[64]) {
                            for (int nn = 0; nn < 8; ++nn)
                                for (int k = 0; k < 4; ++k) {
                                    const int lane = nn * 4 + k;
                                    const double tr = frag[2 * lane], ti = frag[2 * lane + 1];
                                    const double xr = X[2 * slot[k]], xi = X[2 * slot[k] + 1];
                                    acc[nn][0] += tr * xr - ti * xi;
                                    acc[nn][1] += tr * xi + ti * xr;
                                }
                        };
                        if (st.kind == 0) {
                            int e0 = st.w_base[w];
                            for (int jj = 0; jj < j; ++jj) e0 += st.w_count[w * kUnits2 + jj];
                            const int cnt = st.w_count[w * kUnits2 + j];
                            for (int e = e0; e < e0 + cnt; ++e) {
                                int sl[4];
                                for (int k = 0; k < 4; ++k) sl[k] = st.e_slots[4 * e + k] & ~(1 << 30);
                                double fr[64];
                                for (int l = 0; l < 32; ++l) {
                                    fr[2 * l] = st.e_re[32 * e + l];
                                    fr[2 * l + 1] = st.e_im[32 * e + l];
                                }
                                apply(sl, fr);
                            }
                        } else {
                            const int q = st.u_node[u];
                            for (int kt = 0; kt < 2; ++kt) {
                                int slot[4];
                                double frag[64];
                                for (int k = 0; k < 4; ++k) slot[k] = st.u_in[u * 8 + kt * 4 + k];
                                for (int nn = 0; nn < 8; ++nn)
                                    for (int k = 0; k < 4; ++k) {
                                        frag[2 * (nn * 4 + k)] = st.K[2 * (q * 64 + nn * 8 + kt * 4 + k)];
                                        frag[2 * (nn * 4 + k) + 1] = st.K[2 * (q * 64 + nn * 8 + kt * 4 + k) + 1];
                                    }
                                apply(slot, frag);
                            }
                        }
                        for (int nn = 0; nn < 8; ++nn) {
                            const int o = st.u_out[u * 8 + nn];
                            Y[2 * o] = acc[nn][0];
                            Y[2 * o + 1] = acc[nn][1];
                        }
                    }
                std::swap(X, Y);
            }
            std::copy(X.begin(), X.end(), out + 2 * N * b);
        }
    });
}

// Bank-conflict statistics of the compiled v2 tables (host, no GPU): number of
// 16-lane half-warp load / store requests that hit a bank twice.
// Input slots (4 per table entry) of one sparse stage of the compiled v2
// pipeline (profiling / layout experiments). Returns the entry count.
fcct_status fcct_debug_v2_entry_slots(int n, double r, double s, double t, int inverse, int stage, int32_t* out,
                                      int64_t cap, int64_t* count) {
    return guarded([&] {
        auto root = build_tree(n, Params{r, s, t});
        Pipeline2Host h;
        if (!compile_pipeline2(*root, inverse != 0, Shape2{}, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by pipeline v2");
        if (stage < 0 || stage >= static_cast<int>(h.stages.size())) throw FcctError(ST_INVALID_ARGUMENT, "bad stage");
        const auto& st = h.stages[stage];
        *count = static_cast<int64_t>(st.e_slots.size() / 4);
        if (out && cap >= static_cast<int64_t>(st.e_slots.size()))
            std::memcpy(out, st.e_slots.data(), st.e_slots.size() * 4);
    });
}

// Per-stage work of the compiled v2 pipeline (profiling aid): for each stage
// kind, DMMA per tile, the busiest warp's DMMA and the busiest SM sub-partition's
// DMMA (warps w, w+4, w+8, w+12 share one tensor pipe).
fcct_status fcct_debug_v2_stage_stats(int n, double r, double s, double t, int inverse, int64_t* out /* 4*16 */,
                                      int* nstages) {
    return guarded([&] {
        auto root = build_tree(n, Params{r, s, t});
        Pipeline2Host h;
        if (!compile_pipeline2(*root, inverse != 0, Shape2{}, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by pipeline v2");
        const int W = h.shape.warps, U = h.shape.units, MT = h.shape.tb / 4;
        *nstages = static_cast<int>(h.stages.size());
        for (size_t si = 0; si < h.stages.size(); ++si) {
            const auto& st = h.stages[si];
            std::vector<int64_t> per_warp(W, 0);
            for (int w = 0; w < W; ++w) {
                if (st.kind == 0) {
                    for (int e = st.w_base[w]; e < st.w_base[w + 1]; ++e)
                        per_warp[w] += MT * (((st.e_slots[4 * e] >> 30) & 1) ? 2 : 1);
                } else {
                    for (int j = 0; j < U; ++j)
                        if (st.warp_units[w * U + j] >= 0) per_warp[w] += 4 * MT;
                }
            }
            int64_t tot = 0, mx = 0, sp = 0;
            for (int w = 0; w < W; ++w) {
                tot += per_warp[w];
                mx = std::max(mx, per_warp[w]);
            }
            for (int q = 0; q < 4; ++q) {
                int64_t acc = 0;
                for (int w = q; w < W; w += 4) acc += per_warp[w];
                sp = std::max(sp, acc);
            }
            out[4 * si + 0] = st.kind;
            out[4 * si + 1] = tot;
            out[4 * si + 2] = mx;
            out[4 * si + 3] = sp;
            // shared-memory wavefronts of one m-tile's 16-byte accesses (4 lanes
            // k x 2 rows per 8-lane phase; 16-byte bank group = (4 row + slot) mod 8)
            auto wavefronts = [](const int32_t* slots) {
                int64_t wf = 0;
                for (int ph = 0; ph < 4; ++ph) {
                    int cnt[8] = {};
                    for (int rr = 0; rr < 2; ++rr)
                        for (int kk = 0; kk < 4; ++kk) cnt[(4 * (2 * ph + rr) + (slots[kk] & ~(1 << 30))) & 7]++;
                    int m = 0;
                    for (int b = 0; b < 8; ++b) m = std::max(m, cnt[b]);
                    wf += m;
                }
                return wf;
            };
            int64_t ld = 0, ld_ideal = 0, stw = 0, st_ideal = 0;
            if (st.kind == 0) {
                for (size_t e = 0; e < st.e_slots.size() / 4; ++e) {
                    ld += wavefronts(&st.e_slots[4 * e]);
                    ld_ideal += 4;
                }
            } else {
                for (int u = 0; u < st.n_units; ++u)
                    for (int kt = 0; kt < 2; ++kt) {
                        ld += wavefronts(&st.u_in[u * 8 + kt * 4]);
                        ld_ideal += 4;
                    }
            }
            for (int u = 0; u < st.n_units; ++u)
                for (int par = 0; par < 2; ++par) {
                    int32_t sl[4];
                    for (int kk = 0; kk < 4; ++kk) sl[kk] = st.u_out[u * 8 + 2 * kk + par];
                    stw += wavefronts(sl);
                    st_ideal += 4;
                }
            out[64 + 4 * si + 0] = ld;
            out[64 + 4 * si + 1] = ld_ideal;
            out[64 + 4 * si + 2] = stw;
            out[64 + 4 * si + 3] = st_ideal;
        }
    });
}

fcct_status fcct_debug_v2_stats(int n, double r, double s, double t, int inverse, int64_t* stats /* 6 */) {
    return guarded([&] {
        auto root = build_tree(n, Params{r, s, t});
        Pipeline2Host h;
        if (!compile_pipeline2(*root, inverse != 0, Shape2{}, h))
            throw FcctError(ST_INVALID_ARGUMENT, "plan not supported by pipeline v2");
        int64_t ld_req = 0, ld_conf = 0, st_req = 0, st_conf = 0;
        const int stride = h.stride;
        auto conflicted = [&](const int slots[4], bool store) {
            // half-warp lanes 0-15: r = l/4 -> (t_sub, part), k = l%4
            for (int half = 0; half < 2; ++half) {
                bool used[16] = {};
                bool conf = false;
                for (int l = 16 * half; l < 16 * half + 16; ++l) {
                    const int rr = l >> 2, k = l & 3, tsub = rr >> 1, part = rr & 1;
                    const int slot = store ? slots[k] : slots[k];
                    const int bank = ((tsub * stride + 2 * slot + part) % 16 + 16) % 16;
                    if (used[bank]) conf = true;
                    used[bank] = true;
                }
                (store ? st_conf : ld_conf) += conf;
                (store ? st_req : ld_req) += 1;
            }
        };
        for (const auto& st : h.stages)
            for (int u = 0; u < st.n_units; ++u) {
                if (st.kind == 0) {
                    (void)u;
                } else {
                    for (int kt = 0; kt < 2; ++kt) conflicted(&st.u_in[u * 8 + kt * 4], false);
                }
                for (int par = 0; par < 2; ++par) {
                    int sl[4];
                    for (int k = 0; k < 4; ++k) sl[k] = st.u_out[u * 8 + 2 * k + par];
                    conflicted(sl, true);
                }
            }
        for (const auto& st : h.stages)
            if (st.kind == 0)
                for (size_t e = 0; e < st.e_slots.size() / 4; ++e) {
                    int sl[4];
                    for (int k = 0; k < 4; ++k) sl[k] = st.e_slots[4 * e + k] & ~(1 << 30);
                    conflicted(sl, false);
                }
        stats[0] = ld_req;
        stats[1] = ld_conf;
        stats[2] = st_req;
        stats[3] = st_conf;
        stats[4] = h.dmma_per_tile;
        stats[5] = static_cast<int64_t>(h.stages.size());
    });
}

// Profiling aid: per-phase clock64 totals of CTA 0 from the last launch of a
// plan created with FCCT_DEBUG_TIMING set (index 0 = tile load wait,
// 1 + s = stage s). Returns the number of stages.
fcct_status fcct_debug_timing(fcct_plan plan, int inverse, unsigned long long* out, int* nstages) {
    return guarded([&] {
        if (!plan || !plan->v2) throw FcctError(ST_INVALID_ARGUMENT, "plan has no v2 pipeline");
        const auto& t = inverse ? plan->inv2 : plan->fwd2;
        if (!t.desc.timing) throw FcctError(ST_INVALID_ARGUMENT, "FCCT_DEBUG_TIMING was not set at plan creation");
        ck(cudaMemcpy(out, t.desc.timing, sizeof(unsigned long long) * (kMaxStages + 2 + kMaxStages * 16),
                      cudaMemcpyDeviceToHost),
           "D2H");
        *nstages = t.desc.nstages;
    });
}

// Test hook: DMMA fragment-layout probe (device pointers).
fcct_status fcct_debug_dmma_probe(const double* A, const double* B, double* C) {
    return guarded([&] { ck(dmma_probe(A, B, C, nullptr), "dmma probe"); });
}


// ---------------------------------------------------------------------------
// I/O either side of the path (voxel_io.hpp, spectral.cpp)
// ---------------------------------------------------------------------------
namespace {
void copy_string(const std::string& v, char* buf, int64_t len) {
    if (!buf || len <= static_cast<int64_t>(v.size()))
        throw FcctError(ST_INVALID_ARGUMENT, "string buffer too small (need " + std::to_string(v.size() + 1) + " bytes)");
    std::memcpy(buf, v.c_str(), v.size() + 1);
}
std::string path_arg(const char* path) { return path ? std::string(path) : std::string("-"); }
}  // namespace

fcct_status fcct_parse_params(const char* text, double* r, double* s, double* t) {
    return guarded([&] {
        if (!text || !r || !s || !t) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        const Params p = io::parse_params(text);
        *r = p.r;
        *s = p.s;
        *t = p.t;
    });
}

fcct_status fcct_encode_params(double r, double s, double t, char* buf, int64_t len) {
    return guarded([&] { copy_string(io::encode_params(Params{r, s, t}), buf, len); });
}

fcct_status fcct_export_nodes_csv(int n, double r, double s, double t, const char* path) {
    return guarded([&] { io::write_text(path_arg(path), io::nodes_csv(n, Params{r, s, t})); });
}

fcct_status fcct_export_geometry(const char* path) {
    return guarded([&] { io::write_text(path_arg(path), io::geometry_csv()); });
}

fcct_status fcct_export_spectrum(int n, double r, double s, double t, const void* values_host, const char* path) {
    return guarded([&] {
        if (n < 1) throw FcctError(ST_INVALID_ARGUMENT, "skew_nodes: n must be >= 1");
        if (!values_host) throw FcctError(ST_INVALID_ARGUMENT, "null values");
        io::write_text(path_arg(path),
                       io::spectrum_csv(n, Params{r, s, t}, static_cast<const std::complex<double>*>(values_host)));
    });
}

fcct_status fcct_load_spectrum_csv(const char* path, int* n, double* r, double* s, double* t, void* values_host,
                                   int64_t capacity) {
    return guarded([&] {
        if (!path || !n || !r || !s || !t) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        const io::SpectrumFile f = io::load_spectrum_csv(path, values_host == nullptr);
        *n = f.n;
        *r = f.p.r;
        *s = f.p.s;
        *t = f.p.t;
        if (!values_host) return;
        if (capacity < cube(f.n)) throw FcctError(ST_SIZE_MISMATCH, "values buffer holds fewer than n^3 points");
        std::memcpy(values_host, f.values.data(), f.values.size() * sizeof(std::complex<double>));
    });
}

fcct_status fcct_grid_load(const char* path, int* n, double* values_host, int64_t capacity, char* metadata_json,
                           int64_t metadata_len) {
    return guarded([&] {
        if (!path || !n) throw FcctError(ST_INVALID_ARGUMENT, "null argument");
        const io::Grid g = io::load_grid(path);
        *n = g.n;
        if (metadata_json) copy_string(io::metadata_json(g.metadata), metadata_json, metadata_len);
        if (!values_host) return;
        if (capacity < cube(g.n)) throw FcctError(ST_SIZE_MISMATCH, "values buffer holds fewer than n^3 samples");
        std::memcpy(values_host, g.values.data(), g.values.size() * sizeof(double));
    });
}

fcct_status fcct_grid_save(const char* path, int n, const double* values_host, const char* metadata_json) {
    return guarded([&] {
        if (!path) throw FcctError(ST_INVALID_ARGUMENT, "null path");
        if (n < 1) throw FcctError(ST_SIZE_MISMATCH, "grid size must be >= 1");
        if (!values_host) throw FcctError(ST_INVALID_ARGUMENT, "null values");
        io::Grid g;
        g.n = n;
        g.values.assign(values_host, values_host + cube(n));
        g.metadata = io::parse_metadata_json(metadata_json ? metadata_json : "");
        io::save_grid(g, path);
    });
}

fcct_status fcct_synthetic_sword(int n, double* values_host) {
    return guarded([&] {
        if (!values_host) throw FcctError(ST_INVALID_ARGUMENT, "null values");
        const io::Grid g = io::synthetic_sword(n);
        std::memcpy(values_host, g.values.data(), g.values.size() * sizeof(double));
    });
}

fcct_status fcct_occupancy_checksum(const double* values_host, int64_t count, uint64_t* out) {
    return guarded([&] {
        if ((!values_host && count > 0) || !out || count < 0) throw FcctError(ST_INVALID_ARGUMENT, "bad argument");
        *out = io::occupancy_checksum(values_host, count);
    });
}

}  // extern "C"
