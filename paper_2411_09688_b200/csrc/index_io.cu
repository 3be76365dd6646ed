// index_io.cu -- persistence of the offline index (sqz_index_save / _file_info /
// _load).  The paper's offline clustering output is the artefact that is built
// once per fixed context and reused online (section 5 "offline"; P:165-178
// section 3.1); SPEC S:100-103 / S:115-123 names the file magic "SQZIDX1\0" and
// the round-trip property load(save(x)) == x bit-exactly.  The payload is this
// library's own device layout (cluster-major perm + key_off ranges encode the
// membership lists; centroids in the index dtype), not SPEC's per-head ragged
// lists: SPEC binds its CPU program, this file binds the tables sqz.h defines.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/sqz.h"
#include "internal.h"

namespace {

constexpr char MAGIC[8] = {'S', 'Q', 'Z', 'I', 'D', 'X', '1', '\0'};
constexpr uint32_t VERSION = 1;

struct Geom {  // little-endian i64 fields after magic + version
    int64_t H, d, L, levels, c0, c1, c2, dtype, L_total;
};

struct Table {
    void *ptr;
    size_t bytes;
};

// the tables of an index geometry, in file order
std::vector<Table> tables(const sqz_index &x) {
    const size_t H = (size_t)x.H, d = (size_t)x.d, es = x.dtype == SQZ_BF16 ? 2 : 4, i4 = sizeof(int32_t);
    std::vector<Table> t;
    if (x.levels == 3) {
        t.push_back({x.C0, H * x.c0 * d * es});
        t.push_back({x.N0, H * x.c0 * i4});
        t.push_back({x.child_off0, H * ((size_t)x.c0 + 1) * i4});
    }
    if (x.levels >= 2) {
        t.push_back({x.C1, H * x.c1 * d * es});
        t.push_back({x.N1, H * x.c1 * i4});
        t.push_back({x.child_off, H * ((size_t)x.c1 + 1) * i4});
    }
    t.push_back({x.C2, H * x.c2 * d * es});
    t.push_back({x.N2, H * x.c2 * i4});
    t.push_back({x.key_off, H * ((size_t)x.c2 + 1) * i4});
    t.push_back({x.perm, H * (size_t)x.L * i4});
    return t;
}

bool geom_ok(const sqz_index &x) {
    if (x.H < 1 || (x.d != 64 && x.d != 128) || x.L < 1 || x.c2 < 1 || x.c2 > x.L) return false;
    if (x.dtype != SQZ_BF16 && x.dtype != SQZ_F32) return false;
    if (x.levels < 1 || x.levels > 3) return false;
    if (x.levels >= 2 && (x.c1 < 1 || x.c1 > x.c2)) return false;
    if (x.levels == 3 && (x.c0 < 1 || x.c0 > x.c1)) return false;
    if (x.L_total < 0) return false;
    return true;
}

struct File {
    FILE *f = nullptr;
    ~File() {
        if (f) fclose(f);
    }
};

}  // namespace

extern "C" {

int sqz_index_save(const sqz_index *idx, const char *path, void *stream) {
    using sqz::set_error;
    if (!idx || !path) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_save: idx and path are required");
    if (!geom_ok(*idx)) return set_error(SQZ_ERR_FORMAT, "sqz_index_save: invalid index geometry");
    const std::vector<Table> ts = tables(*idx);
    for (const Table &t : ts)
        if (!t.ptr) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_save: a table of the index is NULL");
    File out;
    out.f = fopen(path, "wb");
    if (!out.f) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_save: cannot open %s for writing", path);
    const Geom g{idx->H, idx->d, idx->L, idx->levels, idx->levels == 3 ? idx->c0 : 0,
                 idx->levels >= 2 ? idx->c1 : 0, idx->c2, idx->dtype, idx->L_total};
    bool ok = fwrite(MAGIC, 1, 8, out.f) == 8 && fwrite(&VERSION, sizeof(VERSION), 1, out.f) == 1 &&
              fwrite(&g, sizeof(g), 1, out.f) == 1;
    std::vector<unsigned char> host;
    cudaStream_t st = (cudaStream_t)stream;
    for (const Table &t : ts) {
        if (!ok) break;
        host.resize(t.bytes);
        cudaError_t e = cudaMemcpyAsync(host.data(), t.ptr, t.bytes, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return set_error(SQZ_ERR_CUDA, "sqz_index_save: %s", cudaGetErrorString(e));
        ok = fwrite(host.data(), 1, t.bytes, out.f) == t.bytes;
    }
    if (!ok) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_save: write to %s failed", path);
    return SQZ_OK;
}

int sqz_index_file_info(const char *path, sqz_index *geom) {
    using sqz::set_error;
    if (!path || !geom) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_file_info: path and geom are required");
    File in;
    in.f = fopen(path, "rb");
    if (!in.f) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_file_info: cannot open %s", path);
    char magic[8];
    uint32_t ver = 0;
    Geom g;
    if (fread(magic, 1, 8, in.f) != 8 || std::memcmp(magic, MAGIC, 8) != 0)
        return set_error(SQZ_ERR_FORMAT, "sqz_index_file_info: %s is not a SQZIDX1 index file (bad magic)", path);
    if (fread(&ver, sizeof(ver), 1, in.f) != 1 || ver != VERSION)
        return set_error(SQZ_ERR_FORMAT, "sqz_index_file_info: unsupported SQZIDX1 version %u", ver);
    if (fread(&g, sizeof(g), 1, in.f) != 1)
        return set_error(SQZ_ERR_FORMAT, "sqz_index_file_info: truncated header");
    sqz_index x;
    std::memset(&x, 0, sizeof(x));
    x.H = (int32_t)g.H; x.d = (int32_t)g.d; x.L = g.L; x.levels = (int32_t)g.levels;
    x.c0 = (int32_t)g.c0; x.c1 = (int32_t)g.c1; x.c2 = (int32_t)g.c2; x.dtype = (int32_t)g.dtype;
    x.L_total = g.L_total;
    if (!geom_ok(x)) return set_error(SQZ_ERR_FORMAT, "sqz_index_file_info: invalid geometry in the header");
    // the payload must be exactly the tables of that geometry
    size_t need = 0;
    for (const Table &t : tables(x)) need += t.bytes;
    const long hdr = ftell(in.f);
    if (fseek(in.f, 0, SEEK_END) != 0) return set_error(SQZ_ERR_FORMAT, "sqz_index_file_info: cannot seek");
    const long end = ftell(in.f);
    if (end < 0 || hdr < 0 || (size_t)(end - hdr) != need)
        return set_error(SQZ_ERR_FORMAT, "sqz_index_file_info: payload is %ld bytes, the geometry needs %zu",
                         end - hdr, need);
    *geom = x;
    return SQZ_OK;
}

int sqz_index_load(const char *path, const sqz_index *dst, void *stream) {
    using sqz::set_error;
    if (!dst) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_load: dst is required");
    sqz_index g;
    int rc = sqz_index_file_info(path, &g);
    if (rc) return rc;
    if (g.H != dst->H || g.d != dst->d || g.L != dst->L || g.levels != dst->levels || g.c2 != dst->c2 ||
        g.dtype != dst->dtype || (g.levels >= 2 && g.c1 != dst->c1) || (g.levels == 3 && g.c0 != dst->c0) ||
        g.L_total != dst->L_total)
        return set_error(SQZ_ERR_FORMAT, "sqz_index_load: dst geometry differs from the file's "
                                         "(use sqz_index_file_info to allocate)");
    const std::vector<Table> ts = tables(*dst);
    for (const Table &t : ts)
        if (!t.ptr) return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_load: a table of dst is NULL");
    File in;
    in.f = fopen(path, "rb");
    if (!in.f || fseek(in.f, 8 + sizeof(uint32_t) + sizeof(Geom), SEEK_SET) != 0)
        return set_error(SQZ_ERR_INVALID_ARG, "sqz_index_load: cannot read %s", path);
    std::vector<unsigned char> host;
    cudaStream_t st = (cudaStream_t)stream;
    for (const Table &t : ts) {
        host.resize(t.bytes);
        if (fread(host.data(), 1, t.bytes, in.f) != t.bytes)
            return set_error(SQZ_ERR_FORMAT, "sqz_index_load: truncated payload");
        cudaError_t e = cudaMemcpyAsync(t.ptr, host.data(), t.bytes, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // (host buffer reused)
        if (e != cudaSuccess) return set_error(SQZ_ERR_CUDA, "sqz_index_load: %s", cudaGetErrorString(e));
    }
    return SQZ_OK;
}

}  // extern "C"
