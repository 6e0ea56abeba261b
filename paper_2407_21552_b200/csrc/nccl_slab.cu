// nccl_slab.cu -- the multi-GPU PDM precompute as ONE C-ABI call over an NCCL
// communicator: build_pdm_set (acceleration.py:
// 199-241) over this rank's x-slab of a volume split across the ranks.
//
//   1. slab table: ncclAllGather of every rank's block-plane count (+ an error
//      flag), read back once, so every rank validates the same table and
//      fails together instead of leaving peers inside a collective;
//   2. range_apron: neighbours swap one boundary voxel plane (ncclSend/Recv:
//      x is the slowest axis, so a plane is one contiguous ny*nz run) and fold
//      its apron min/max into the first/last block plane;
//   3. the partition mask, then the 1-D distance along x (the shard axis)
//      inside the slab;
//   4. ncclAllGather of every slab's two edge planes per partition
//      (2 * n * by * bz bytes per rank, 16.8 MB per rank at 2048^3 / 8 GPUs
//      instead of a 254-plane halo), fold of the other slabs' nearest occupied
//      blocks (bit-exact: a min of clamped distances), the local y/z passes;
//   5. the merge's packed planes.
//
// Everything is enqueued on the caller's stream (NCCL runs on it too); the
// call synchronises once, for the slab table.  NCCL is resolved at run time
// (dlopen of libnccl.so.2 -- inside a torch process that is torch's own
// already-loaded NCCL, so a communicator from ProcessGroupNCCL._comm_ptr()
// works), so the library itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "pdm_common.cuh"

namespace pdm {
namespace {

struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
};

const Nccl &nccl() {
    static Nccl api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
#define PDM_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
        PDM_NCCL_SYM(get_unique_id, "ncclGetUniqueId");
        PDM_NCCL_SYM(comm_init_rank, "ncclCommInitRank");
        PDM_NCCL_SYM(comm_destroy, "ncclCommDestroy");
        PDM_NCCL_SYM(comm_count, "ncclCommCount");
        PDM_NCCL_SYM(comm_user_rank, "ncclCommUserRank");
        PDM_NCCL_SYM(all_gather, "ncclAllGather");
        PDM_NCCL_SYM(send, "ncclSend");
        PDM_NCCL_SYM(recv, "ncclRecv");
        PDM_NCCL_SYM(group_start, "ncclGroupStart");
        PDM_NCCL_SYM(group_end, "ncclGroupEnd");
        PDM_NCCL_SYM(error_string, "ncclGetErrorString");
#undef PDM_NCCL_SYM
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count &&
                 api.comm_user_rank && api.all_gather && api.send && api.recv &&
                 api.group_start && api.group_end && api.error_string;
    });
    return api;
}

#define PDM_NCCL_TRY(expr)                                                                   \
    do {                                                                                     \
        ncclResult_t r_ = (expr);                                                            \
        if (r_ != ncclSuccess) {                                                             \
            ::pdm::set_error("%s failed: %s (%s:%d)", #expr, nccl().error_string(r_), __FILE__, \
                             __LINE__);                                                      \
            return PDM_ECUDA;                                                                \
        }                                                                                    \
    } while (0)

#define PDM_NCCL_REQUIRE()                                                                 \
    PDM_REQUIRE(nccl().ok, "NCCL is not available (libnccl.so.2 could not be loaded)")

constexpr int64_t kAlign = 256;

struct Layout {  // byte offsets of the workspace pieces
    int64_t table, mask, mins, maxs, plane_lo, plane_hi, pm_lo, px_lo, pm_hi, px_hi, edges,
        edges_all, total;
};

Layout layout(int world, int bits, int64_t nx, int64_t ny, int64_t nz, int b, int n) {
    const int64_t vb = bits == 8 ? 1 : 2;
    const int64_t bx = ceil_div(nx, b), by = ceil_div(ny, b), bz = ceil_div(nz, b);
    const int64_t nb = bx * by * bz, words = (n + 31) / 32;
    Layout L{};
    int64_t at = 0;
    auto take = [&](int64_t bytes) {
        const int64_t o = at;
        at += ceil_div(bytes, kAlign) * kAlign;
        return o;
    };
    L.table = take(8 * 2 * (int64_t)world);
    L.mask = take(4 * nb * words);
    L.mins = take(vb * nb);
    L.maxs = take(vb * nb);
    L.plane_lo = take(vb * ny * nz);
    L.plane_hi = take(vb * ny * nz);
    L.pm_lo = take(vb * by * bz);
    L.px_lo = take(vb * by * bz);
    L.pm_hi = take(vb * by * bz);
    L.px_hi = take(vb * by * bz);
    L.edges = take(2 * (int64_t)n * by * bz);
    L.edges_all = take(2 * (int64_t)n * by * bz * world);
    L.total = at;
    return L;
}

}  // namespace
}  // namespace pdm

using namespace pdm;

extern "C" int pdm_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int pdm_nccl_unique_id(uint8_t *id_out) {
    PDM_NCCL_REQUIRE();
    PDM_REQUIRE(id_out, "pdm_nccl_unique_id: null pointer");
    ncclUniqueId id;
    PDM_NCCL_TRY(nccl().get_unique_id(&id));
    memcpy(id_out, id.internal, sizeof(id.internal));
    return PDM_OK;
}

extern "C" int pdm_nccl_comm_init(void **comm_out, int32_t world, const uint8_t *id, int32_t rank) {
    PDM_NCCL_REQUIRE();
    PDM_REQUIRE(comm_out && id && world >= 1 && rank >= 0 && rank < world,
                "pdm_nccl_comm_init: bad arguments");
    ncclUniqueId uid;
    memcpy(uid.internal, id, sizeof(uid.internal));
    ncclComm_t c = nullptr;
    PDM_NCCL_TRY(nccl().comm_init_rank(&c, world, uid, rank));
    *comm_out = c;
    return PDM_OK;
}

extern "C" int pdm_nccl_comm_count(void *comm) {
    if (!nccl().ok || !comm) return -1;
    int world = 0;
    if (nccl().comm_count(static_cast<ncclComm_t>(comm), &world) != ncclSuccess) return -1;
    return world;
}

extern "C" int pdm_nccl_comm_destroy(void *comm) {
    PDM_NCCL_REQUIRE();
    if (comm) PDM_NCCL_TRY(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
    return PDM_OK;
}

extern "C" int64_t pdm_build_pdm_set_slab_nccl_workspace(int32_t world, int bits, int64_t nx,
                                                         int64_t ny, int64_t nz, int32_t b,
                                                         int32_t n) {
    if (world < 1 || (bits != 8 && bits != 16) || nx < 1 || ny < 1 || nz < 1 || b < 1 || n < 1)
        return -1;
    return layout(world, bits, nx, ny, nz, b, n).total;
}

extern "C" int pdm_build_pdm_set_slab_nccl(void *comm, const void *vox, int bits, int64_t nx,
                                           int64_t ny, int64_t nz, int32_t b,
                                           const int32_t *pid, int32_t n, int32_t mode,
                                           int64_t bx0_expected, uint8_t *pdms,
                                           int64_t plane_pitch, uint8_t *nib, int64_t nib_pitch,
                                           uint8_t *base, int64_t base_pitch,
                                           uint32_t *violations, void *workspace,
                                           int64_t workspace_bytes, int64_t *slab_out,
                                           pdm_stream_t stream) {
    const char *fn = "pdm_build_pdm_set_slab_nccl";
    PDM_NCCL_REQUIRE();
    PDM_REQUIRE(comm && vox && pid && pdms && workspace && slab_out, "%s: null pointer", fn);
    PDM_REQUIRE(mode == 0 || mode == 1, "%s: mode must be 0 (voxel) or 1 (range_apron)", fn);
    PDM_REQUIRE(bits == 8 || bits == 16, "%s: bits must be 8 or 16", fn);
    PDM_REQUIRE(!nib || (base && violations), "%s: packed planes need base and violations", fn);
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int world = 0, rank = 0;
    PDM_NCCL_TRY(nccl().comm_count(c, &world));
    PDM_NCCL_TRY(nccl().comm_user_rank(c, &rank));
    const Layout L = layout(world, bits, nx, ny, nz, b, n);
    PDM_REQUIRE(workspace_bytes >= L.total, "%s: workspace of %lld bytes needs %lld", fn,
                (long long)workspace_bytes, (long long)L.total);
    cudaStream_t s = as_stream(stream);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    const int64_t vb = bits == 8 ? 1 : 2;
    const int64_t bx = ceil_div(nx, b), by = ceil_div(ny, b), bz = ceil_div(nz, b);
    const int64_t nb = bx * by * bz;
    const int words = (n + 31) / 32;

    // 1. slab table: (block planes, "ends inside a block") of every rank
    int64_t mine[2] = {bx, nx % b != 0 ? 1 : 0};
    int64_t *table_d = reinterpret_cast<int64_t *>(ws + L.table);
    PDM_CUDA_TRY(cudaMemcpyAsync(table_d + 2 * rank, mine, sizeof(mine), cudaMemcpyHostToDevice,
                                 s));
    PDM_NCCL_TRY(nccl().all_gather(table_d + 2 * rank, table_d, 2, ncclInt64, c, s));
    std::vector<int64_t> table(2 * (size_t)world);
    PDM_CUDA_TRY(cudaMemcpyAsync(table.data(), table_d, table.size() * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s));
    PDM_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int64_t> starts(world + 1, 0);
    for (int r = 0; r < world; ++r) starts[r + 1] = starts[r] + table[2 * r];
    for (int r = 0; r + 1 < world; ++r)
        PDM_REQUIRE(!table[2 * r + 1], "%s: rank %d: only the last slab may end inside a block",
                    fn, r);
    PDM_REQUIRE(bx0_expected < 0 || bx0_expected == starts[rank],
                "%s: rank %d: slab starts at block %lld, expected %lld", fn, rank,
                (long long)bx0_expected, (long long)starts[rank]);
    slab_out[0] = starts[rank];
    slab_out[1] = starts[rank + 1];
    slab_out[2] = starts[world];

    // 2-3. partition mask (range_apron: with the neighbours' boundary planes)
    uint32_t *mask = reinterpret_cast<uint32_t *>(ws + L.mask);
    int st;
    if (mode == 0) {
        st = pdm_partition_mask_voxel(vox, bits, nx, ny, nz, b, pid, n, mask, words, stream);
        if (st) return st;
    } else {
        const int64_t plane = ny * nz;
        const uint8_t *v8 = static_cast<const uint8_t *>(vox);
        uint8_t *lo = ws + L.plane_lo, *hi = ws + L.plane_hi;
        PDM_NCCL_TRY(nccl().group_start());
        if (rank > 0) {
            PDM_NCCL_TRY(nccl().send(v8, plane * vb, ncclUint8, rank - 1, c, s));
            PDM_NCCL_TRY(nccl().recv(lo, plane * vb, ncclUint8, rank - 1, c, s));
        }
        if (rank < world - 1) {
            PDM_NCCL_TRY(nccl().send(v8 + (nx - 1) * plane * vb, plane * vb, ncclUint8, rank + 1,
                                     c, s));
            PDM_NCCL_TRY(nccl().recv(hi, plane * vb, ncclUint8, rank + 1, c, s));
        }
        PDM_NCCL_TRY(nccl().group_end());
        void *mins = ws + L.mins, *maxs = ws + L.maxs;
        if ((st = pdm_block_min_max(vox, bits, nx, ny, nz, b, mins, maxs, stream))) return st;
        const int64_t bplane = by * bz;
        if (rank > 0) {
            if ((st = pdm_block_min_max(lo, bits, 1, ny, nz, b, ws + L.pm_lo, ws + L.px_lo,
                                        stream)) ||
                (st = pdm_minmax_fold(mins, maxs, ws + L.pm_lo, ws + L.px_lo, bits, bplane,
                                      stream)))
                return st;
        }
        if (rank < world - 1) {
            uint8_t *mn_last = static_cast<uint8_t *>(mins) + (bx - 1) * bplane * vb;
            uint8_t *mx_last = static_cast<uint8_t *>(maxs) + (bx - 1) * bplane * vb;
            if ((st = pdm_block_min_max(hi, bits, 1, ny, nz, b, ws + L.pm_hi, ws + L.px_hi,
                                        stream)) ||
                (st = pdm_minmax_fold(mn_last, mx_last, ws + L.pm_hi, ws + L.px_hi, bits, bplane,
                                      stream)))
                return st;
        }
        if ((st = pdm_partition_mask_minmax(mins, maxs, bits, nb, pid, n, mask, words, stream)))
            return st;
    }
    if ((st = pdm_dt_pass_x_mask(mask, words, n, bx, by, bz, pdms, plane_pitch, stream)))
        return st;

    // 4. edge planes of every slab, fold, local y / z passes
    uint8_t *edges = ws + L.edges, *edges_all = ws + L.edges_all;
    const int64_t ebytes = 2 * (int64_t)n * by * bz;
    if ((st = pdm_dt_slab_edges(pdms, plane_pitch, n, bx, by, bz, edges, stream))) return st;
    PDM_NCCL_TRY(nccl().all_gather(edges, edges_all, ebytes, ncclUint8, c, s));
    if ((st = pdm_dt_slab_fold(pdms, plane_pitch, n, bx, by, bz, edges_all, world, rank,
                               starts.data(), stream)))
        return st;
    if ((st = pdm_dt_pass_yz(pdms, plane_pitch, n, bx, by, bz, stream))) return st;

    // 5. the merge's packed planes
    if (nib)
        return pdm_pack_pdms(pdms, plane_pitch, nb, n, nib, nib_pitch, base, base_pitch,
                             violations, stream);
    return PDM_OK;
}
