// dist.cu -- multi-GPU entry points of the C ABI: the host-side shard plan,
// the shard-index builder and the NCCL communicator (resolved at run time, so
// libsqz itself has no link-time NCCL dependency and loads on any host).
//
// Cluster sharding: every rank holds the clusters p with
// p mod world == rank (Level-1 subtrees intact) and their keys.  The lookup's
// per-query (m, D) statistics are all-gathered once per level so that every
// rank thresholds against the global Eq. 1 / Eq. 3 denominator; the attention
// partials (O, LSE) are all-gathered and merged in rank order.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/sqz.h"
#include "internal.h"

using namespace sqz;

namespace {

// ---------------------------------------------------------------- NCCL table
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    // point-to-point (the head-slice exchange); optional
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    bool ok = false;
    char why[256] = "";
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // prefer the copy already in the process (torch's), else the system one
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.why, sizeof(api.why), "cannot load libnccl.so.2: %s", dlerror());
            return;
        }
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
        api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
        api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
        api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
                 api.GetErrorString;
        if (!api.ok) snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks a required symbol");
    });
    return api;
}

struct Comm {
    ncclComm_t c;
    int rank, world;
};

int nccl_fail(ncclResult_t r, const char *what) {
    return set_error(SQZ_ERR_NCCL, "%s: %s", what, nccl().GetErrorString(r));
}

}  // namespace

namespace sqz {
int comm_world(void *comm) { return comm ? static_cast<Comm *>(comm)->world : 1; }

// all-gather of `count` floats per rank: recv [world, count]
int comm_allgather_f32(void *comm, const float *send, float *recv, size_t count, cudaStream_t st) {
    Comm *c = static_cast<Comm *>(comm);
    ncclResult_t r = nccl().AllGather(send, recv, count, ncclFloat32, c->c, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    return SQZ_OK;
}
}  // namespace sqz

extern "C" {

// ------------------------------------------------------------------ shard plan
int sqz_shard_plan_compute(int32_t H, int32_t levels, int32_t c1, int32_t c2, int64_t L,
                           const int32_t *key_off, const int32_t *child_off, int32_t rank,
                           int32_t world, sqz_shard_plan *plan) {
    if (!plan) return set_error(SQZ_ERR_INVALID_ARG, "plan is NULL");
    if (H < 1 || c2 < 1 || L < 1) return set_error(SQZ_ERR_INVALID_ARG, "H, c2, L must be >= 1");
    if (levels != 1 && levels != 2) return set_error(SQZ_ERR_INVALID_ARG, "levels must be 1 or 2");
    if (world < 1 || rank < 0 || rank >= world)
        return set_error(SQZ_ERR_INVALID_ARG, "rank = %d, world = %d: need 0 <= rank < world", rank,
                         world);
    if (!key_off) return set_error(SQZ_ERR_INVALID_ARG, "key_off is NULL");
    if (levels == 2 && (!child_off || c1 < 1))
        return set_error(SQZ_ERR_INVALID_ARG, "levels == 2 needs child_off and c1 >= 1");
    const int top = levels == 2 ? c1 : c2;  // the sharded level
    if (top < world)
        return set_error(SQZ_ERR_INVALID_ARG, "%d clusters at the sharded level < world = %d", top,
                         world);
    // owned top-level clusters (same count in every head)
    const int n_top = (top - rank + world - 1) / world;
    // per head: local Level-2 clusters (global ids, in order) and keys
    std::vector<std::vector<int32_t>> l2(H);
    int32_t c2_loc = 0;
    int64_t L_loc = 0;
    for (int h = 0; h < H; ++h) {
        const int32_t *ko = key_off + (size_t)h * (c2 + 1);
        if (ko[0] != 0 || ko[c2] > L) return set_error(SQZ_ERR_INVALID_ARG, "key_off[%d] inconsistent", h);
        int64_t keys = 0;
        for (int j = 0; j < n_top; ++j) {
            const int p = rank + j * world;
            int a = p, b = p + 1;
            if (levels == 2) {
                const int32_t *co = child_off + (size_t)h * (c1 + 1);
                a = co[p];
                b = co[p + 1];
                if (a < 0 || b < a || b > c2)
                    return set_error(SQZ_ERR_INVALID_ARG, "child_off[%d][%d] inconsistent", h, p);
            }
            for (int i = a; i < b; ++i) {
                if (ko[i + 1] < ko[i]) return set_error(SQZ_ERR_INVALID_ARG, "key_off[%d] decreasing", h);
                l2[h].push_back(i);
                keys += ko[i + 1] - ko[i];
            }
        }
        c2_loc = std::max<int32_t>(c2_loc, (int32_t)l2[h].size());
        L_loc = std::max<int64_t>(L_loc, keys);
    }
    plan->c1 = levels == 2 ? n_top : 0;
    plan->c2 = std::max<int32_t>(c2_loc, 1);
    plan->L = std::max<int64_t>(L_loc, 1);
    const int32_t C1 = plan->c1, C2 = plan->c2;
    const int64_t LL = plan->L;
    for (int h = 0; h < H; ++h) {
        const int32_t *ko = key_off + (size_t)h * (c2 + 1);
        const int n2 = (int)l2[h].size();
        if (levels == 2) {
            const int32_t *co = child_off + (size_t)h * (c1 + 1);
            int run = 0;
            for (int j = 0; j < C1; ++j) {
                const int p = rank + j * world;
                if (plan->c1_src) plan->c1_src[(size_t)h * C1 + j] = p;
                const int nch = co[p + 1] - co[p];
                if (plan->child_off) plan->child_off[(size_t)h * (C1 + 1) + j] = run;
                if (plan->N1) plan->N1[(size_t)h * C1 + j] = ko[co[p + 1]] - ko[co[p]];
                run += nch;
            }
            if (plan->child_off) plan->child_off[(size_t)h * (C1 + 1) + C1] = run;
        }
        int64_t pos = 0;
        for (int i = 0; i < C2; ++i) {
            const int g = i < n2 ? l2[h][i] : -1;
            const int n = g >= 0 ? ko[g + 1] - ko[g] : 0;
            if (plan->c2_src) plan->c2_src[(size_t)h * C2 + i] = g;
            if (plan->N2) plan->N2[(size_t)h * C2 + i] = n;
            if (plan->key_off) plan->key_off[(size_t)h * (C2 + 1) + i] = (int32_t)pos;
            if (plan->key_src)
                for (int t = 0; t < n; ++t) plan->key_src[(size_t)h * LL + pos + t] = ko[g] + t;
            pos += n;
        }
        if (plan->key_off) plan->key_off[(size_t)h * (C2 + 1) + C2] = (int32_t)pos;
        if (plan->key_src)
            for (int64_t t = pos; t < LL; ++t) plan->key_src[(size_t)h * LL + t] = -1;
    }
    return SQZ_OK;
}

int sqz_index_shard(const sqz_index *full, const void *Kp, const void *Vp, const int32_t *c1_src,
                    const int32_t *c2_src, const int32_t *key_src, const sqz_index *local,
                    void *Kp_local, void *Vp_local, void *stream) {
    if (!full || !local) return set_error(SQZ_ERR_INVALID_ARG, "full / local is NULL");
    if (!Kp || !Vp || !Kp_local || !Vp_local || !c2_src || !key_src)
        return set_error(SQZ_ERR_INVALID_ARG, "Kp, Vp, Kp_local, Vp_local, c2_src, key_src required");
    if (!full->C2 || !local->C2 || !local->perm)
        return set_error(SQZ_ERR_INVALID_ARG, "full->C2, local->C2, local->perm required");
    if (local->H != full->H || local->d != full->d || local->dtype != full->dtype ||
        local->levels != full->levels)
        return set_error(SQZ_ERR_INVALID_ARG, "local geometry (H, d, dtype, levels) must match full");
    if (full->levels == 2 && (!c1_src || !full->C1 || !local->C1))
        return set_error(SQZ_ERR_INVALID_ARG, "levels == 2 needs c1_src, full->C1, local->C1");
    cudaError_t e = launch_shard_gather(*full, Kp, Vp, c1_src, c2_src, key_src, *local, Kp_local,
                                        Vp_local, (cudaStream_t)stream);
    if (e != cudaSuccess) return set_error(SQZ_ERR_CUDA, "shard gather: %s", cudaGetErrorString(e));
    return SQZ_OK;
}

// ------------------------------------------------------------------ comm
int sqz_comm_unique_id(uint8_t id[128]) {
    if (!id) return set_error(SQZ_ERR_INVALID_ARG, "id is NULL");
    if (!nccl().ok) return set_error(SQZ_ERR_NCCL, "%s", nccl().why);
    ncclUniqueId u;
    ncclResult_t r = nccl().GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
    return SQZ_OK;
}

int sqz_comm_init(const uint8_t id[128], int32_t rank, int32_t world, void **comm) {
    if (!id || !comm) return set_error(SQZ_ERR_INVALID_ARG, "id / comm is NULL");
    if (world < 1 || rank < 0 || rank >= world)
        return set_error(SQZ_ERR_INVALID_ARG, "rank = %d, world = %d", rank, world);
    if (!nccl().ok) return set_error(SQZ_ERR_NCCL, "%s", nccl().why);
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    Comm *c = new Comm{nullptr, rank, world};
    ncclResult_t r = nccl().CommInitRank(&c->c, world, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *comm = c;
    return SQZ_OK;
}

int sqz_comm_destroy(void *comm) {
    if (!comm) return SQZ_OK;
    Comm *c = static_cast<Comm *>(comm);
    ncclResult_t r = nccl().CommDestroy(c->c);
    delete c;
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return SQZ_OK;
}

int sqz_comm_merge_workspace(int32_t world, int64_t rows, int32_t d, size_t *ws_bytes) {
    if (world < 1 || rows < 0 || d < 1 || !ws_bytes)
        return set_error(SQZ_ERR_INVALID_ARG, "world >= 1, rows >= 0, d >= 1, ws_bytes required");
    *ws_bytes = (size_t)world * rows * (d + 1) * sizeof(float) + 1024;
    return SQZ_OK;
}

int sqz_comm_allgather_merge(void *comm, const float *O_part, const float *LSE_part, int64_t rows,
                             int32_t d, void *O, float *LSE, int32_t out_dtype, void *ws,
                             size_t ws_bytes, void *stream) {
    if (!comm) return set_error(SQZ_ERR_INVALID_ARG, "comm is NULL");
    if (!O_part || !LSE_part || !O || !LSE || !ws)
        return set_error(SQZ_ERR_INVALID_ARG, "O_part, LSE_part, O, LSE, ws required");
    if (rows < 0 || rows > 0x7fffffffLL || d < 1)
        return set_error(SQZ_ERR_INVALID_ARG, "rows in [0, 2^31) and d >= 1 required");
    if (out_dtype != SQZ_F32 && out_dtype != SQZ_BF16)
        return set_error(SQZ_ERR_INVALID_ARG, "out_dtype = %d is not a sqz_dtype", out_dtype);
    Comm *c = static_cast<Comm *>(comm);
    size_t need = 0;
    sqz_comm_merge_workspace(c->world, rows, d, &need);
    if (ws_bytes < need) return set_error(SQZ_ERR_INVALID_ARG, "ws_bytes = %zu < %zu", ws_bytes, need);
    char *base = reinterpret_cast<char *>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float *Og = reinterpret_cast<float *>(base);
    float *Lg = Og + (size_t)c->world * rows * d;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = comm_allgather_f32(comm, O_part, Og, (size_t)rows * d, st);
    if (rc) return rc;
    rc = comm_allgather_f32(comm, LSE_part, Lg, (size_t)rows, st);
    if (rc) return rc;
    cudaError_t e = launch_merge(c->world, Og, Lg, rows, d, O, LSE, out_dtype, st);
    if (e != cudaSuccess) return set_error(SQZ_ERR_CUDA, "merge launch: %s", cudaGetErrorString(e));
    return SQZ_OK;
}

int sqz_comm_alltoall_merge_workspace(int32_t world, int32_t B, int32_t H, int32_t n_q, int32_t d,
                                      size_t *ws_bytes) {
    if (world < 1 || B < 1 || H < 1 || n_q < 1 || d < 1 || !ws_bytes)
        return set_error(SQZ_ERR_INVALID_ARG, "world, B, H, n_q, d >= 1 and ws_bytes required");
    if (H % world) return set_error(SQZ_ERR_INVALID_ARG, "H = %d is not a multiple of world = %d", H, world);
    const size_t rows = (size_t)B * (H / world) * n_q;
    *ws_bytes = (size_t)world * rows * (d + 1) * sizeof(float) + 1024;
    return SQZ_OK;
}

int sqz_comm_alltoall_merge(void *comm, const float *O_part, const float *LSE_part, int32_t B, int32_t H,
                            int32_t n_q, int32_t d, void *O_slice, float *LSE_slice, int32_t out_dtype,
                            void *ws, size_t ws_bytes, void *stream) {
    if (!comm) return set_error(SQZ_ERR_INVALID_ARG, "comm is NULL");
    if (!O_part || !LSE_part || !O_slice || !LSE_slice || !ws)
        return set_error(SQZ_ERR_INVALID_ARG, "O_part, LSE_part, O_slice, LSE_slice, ws required");
    if (out_dtype != SQZ_F32 && out_dtype != SQZ_BF16)
        return set_error(SQZ_ERR_INVALID_ARG, "out_dtype = %d is not a sqz_dtype", out_dtype);
    Comm *c = static_cast<Comm *>(comm);
    size_t need = 0;
    int rc = sqz_comm_alltoall_merge_workspace(c->world, B, H, n_q, d, &need);
    if (rc) return rc;
    if (ws_bytes < need) return set_error(SQZ_ERR_INVALID_ARG, "ws_bytes = %zu < %zu", ws_bytes, need);
    NcclApi &api = nccl();
    if (!api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd)
        return set_error(SQZ_ERR_NCCL, "libnccl.so.2 lacks ncclSend / ncclRecv / ncclGroupStart / ncclGroupEnd");
    const int W = c->world, Hs = H / W;
    const size_t rows = (size_t)B * Hs * n_q, blk = (size_t)Hs * n_q;  // rows of one (b, head slice)
    char *base = reinterpret_cast<char *>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float *Or = reinterpret_cast<float *>(base);  // [W][B][Hs][n_q][d] (merge layout [P][rows][d])
    float *Lr = Or + (size_t)W * rows * d;        // [W][B][Hs][n_q]
    cudaStream_t st = (cudaStream_t)stream;
    ncclResult_t r = api.GroupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    for (int p = 0; p < W && r == ncclSuccess; ++p)
        for (int b = 0; b < B && r == ncclSuccess; ++b) {
            // my partial rows of peer p's heads, and peer p's partial rows of my heads
            const size_t src = ((size_t)b * H + (size_t)p * Hs) * n_q;
            const size_t dst = ((size_t)p * B + b) * blk;
            r = api.Send(O_part + src * d, blk * d, ncclFloat32, p, c->c, st);
            if (r == ncclSuccess) r = api.Recv(Or + dst * d, blk * d, ncclFloat32, p, c->c, st);
            if (r == ncclSuccess) r = api.Send(LSE_part + src, blk, ncclFloat32, p, c->c, st);
            if (r == ncclSuccess) r = api.Recv(Lr + dst, blk, ncclFloat32, p, c->c, st);
        }
    const ncclResult_t r2 = api.GroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
    cudaError_t e = launch_merge(W, Or, Lr, (int64_t)rows, d, O_slice, LSE_slice, out_dtype, st);
    if (e != cudaSuccess) return set_error(SQZ_ERR_CUDA, "merge launch: %s", cudaGetErrorString(e));
    return SQZ_OK;
}

}  // extern "C"
