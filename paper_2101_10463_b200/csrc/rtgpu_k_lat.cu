/* rtgpu_k_lat.cu -- the lattice path's kernel (lattice.cuh): exact FP64
 * verdicts and end-to-end bounds with per-task scales, for any SM count. */
#include "kernel.cuh"
#include "lattice.cuh"

namespace rtgpu {

/* Persistent teams of W warps, one task set each (256 threads per CTA, 8 / W
 * teams, team t on named barrier t + 1).  LIST = false: the sets
 * [set_base, set_base + n_sets) (the front stage of bounds runs); LIST =
 * true: the sets the fast kernel handed on in esc[0] (verdict runs), whose
 * decided entries become -1.  Sets the path does not take go on to esc[0]
 * (front) or stay in it (list) for the general stages. */
/* MINB: 256-thread CTAs per SM the register allocation must allow -- 4 (64
 * registers, 32 warps) for small slabs, 2 (128 registers, no spills in the
 * fixed-point loop, 16 warps) when shared memory caps residency anyway. */
#ifndef RTGPU_LAT_THREADS
#define RTGPU_LAT_THREADS 256 /* CTA size: RTGPU_LAT_THREADS / 32 / W teams per CTA */
#endif

template <int W, bool LIST, int MINB>
__global__ void __launch_bounds__(RTGPU_LAT_THREADS, MINB) lattice_kernel(KParams p, int slab_bytes) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int team = warp / W;
    LTeam<W> tm{lane, warp % W, team + 1};
    LCtx c;
    c.hbase = nullptr;
    c.sto = LSLAB_HDR + warp * LST_BYTES;
    c.base = LSLAB_HDR + (RTGPU_LAT_THREADS / 32) * LST_BYTES + team * slab_bytes;
    if (threadIdx.x == 0) {
        LSlab L;
        L.init(p.dims);
        *(LSlab *)rt_dyn_smem = L;
    }
    __syncthreads();
    const bool bounds = (p.flags & RTGPU_F_BOUNDS) != 0;
    const i64 count = LIST ? (i64)p.ctr[4] : p.n_sets;
    unsigned long long *wctr = LIST ? p.lat_ctr : p.wctr0;
    i64 *slot = (i64 *)(rt_dyn_smem + c.base + c.L().o_red) + 16; /* the team's set index */
    for (;;) {
        if (tm.leader()) *slot = (i64)atomicAdd(wctr, 1ull);
        tm.sync();
        const i64 idx = *slot;
        tm.sync();
        if (idx >= count) break;
        const i64 s = LIST ? p.esc[0][idx] : p.set_base + idx;
        if (s < 0) continue;
        c.blob = p.blobs + p.set_off[s];
        /* list stage: the sets the fast path could not take because of their
         * width (more than 64 SMs); its range escalations (a few per 10^5 on
         * 10 SMs) stay with the int64 fast path, which decides them sooner */
        if (LIST && c.blob[1] <= 64 && c.blob[7] >= 1) continue;
        const i64 tb = p.task_base[s];
        i64 evals = 0;
        const int st = lattice_set(tm, c, bounds, p.vsm + tb, bounds ? p.e2e + tb : nullptr,
                                   bounds ? p.den + tb : nullptr, evals);
        if (st == ST_ESCALATE) {
            if (!LIST && tm.leader()) {
                unsigned long long pos = atomicAdd(&p.ctr[4], 1ull);
                p.esc[0][pos] = s;
            }
            tm.sync();
            continue;
        }
        if (tm.leader()) {
            p.status[s] = st;
            p.evals[s] = evals;
            if (LIST) p.esc[0][idx] = -1;
        }
        tm.sync();
    }
}

/* Kernel shape from the slab size (measured, scripts/gpu_lat_ab.sh r2d:
 * barriers and spills cost more than occupancy): one warp per set while
 * 16 slabs fit (32 warps at 64 registers when 32 slabs fit, else 16 warps at
 * 128), else teams of 2 (or 4) warps at 128 registers. */
#ifndef RTGPU_LAT_SMALL_MINB
#define RTGPU_LAT_SMALL_MINB 2
#endif
#ifndef RTGPU_LAT_MED_MINB
#define RTGPU_LAT_MED_MINB 2
#endif
struct LatShape {
    int W, minb;
};
static LatShape lat_shape(const LSlab &L) {
    const int cap = 220 * 1024, wpc = RTGPU_LAT_THREADS / 32; /* warps per CTA */
    if (L.bytes * wpc * RTGPU_LAT_SMALL_MINB <= cap) return {1, RTGPU_LAT_SMALL_MINB};
    if (L.bytes * wpc * RTGPU_LAT_MED_MINB <= cap) return {1, RTGPU_LAT_MED_MINB};
    if (L.bytes * 16 <= cap) return {1, RTGPU_LAT_MED_MINB};
    if (L.bytes * 8 <= cap) return {2, RTGPU_LAT_MED_MINB};
    return {4, RTGPU_LAT_MED_MINB};
}

template <int W, bool LIST, int MINB> static void *lat_kernel_ptr() { return (void *)lattice_kernel<W, LIST, MINB>; }
static void *lat_kernel_for(LatShape sh, bool list) {
    if (sh.W == 1 && sh.minb == RTGPU_LAT_SMALL_MINB)
        return list ? lat_kernel_ptr<1, true, RTGPU_LAT_SMALL_MINB>() : lat_kernel_ptr<1, false, RTGPU_LAT_SMALL_MINB>();
    if (sh.W == 1 && sh.minb == RTGPU_LAT_MED_MINB)
        return list ? lat_kernel_ptr<1, true, RTGPU_LAT_MED_MINB>() : lat_kernel_ptr<1, false, RTGPU_LAT_MED_MINB>();
    if (sh.W == 2)
        return list ? lat_kernel_ptr<2, true, RTGPU_LAT_MED_MINB>() : lat_kernel_ptr<2, false, RTGPU_LAT_MED_MINB>();
    return list ? lat_kernel_ptr<4, true, RTGPU_LAT_MED_MINB>() : lat_kernel_ptr<4, false, RTGPU_LAT_MED_MINB>();
}

static int lat_launch(const KParams &p, bool list, cudaStream_t st) {
    LSlab L;
    L.init(p.dims);
    const LatShape sh = lat_shape(L);
    const int W = sh.W;
    const int teams = RTGPU_LAT_THREADS / 32 / W;
    const int bytes = LSLAB_HDR + (RTGPU_LAT_THREADS / 32) * LST_BYTES + L.bytes * teams;
    if (bytes > 227 * 1024) {
        set_err_msg("task sets too large for shared memory");
        return -3;
    }
    void *k = lat_kernel_for(sh, list);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) {
        set_err("cudaFuncSetAttribute", e);
        return -4;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, RTGPU_LAT_THREADS, bytes);
    if (per_sm < 1) per_sm = 1;
    i64 grid = (i64)sms * per_sm;
    if (!list) {
        const i64 want = (p.n_sets + teams - 1) / teams;
        if (want < grid) grid = want;
    }
    if (grid < 1) grid = 1;
    int sb = L.bytes;
    void *args[] = {(void *)&p, (void *)&sb};
    e = cudaLaunchKernel(k, dim3((unsigned)grid), dim3(RTGPU_LAT_THREADS), args, bytes, st);
    count_launch();
    if (e != cudaSuccess) {
        set_err("lattice_kernel launch", e);
        return -5;
    }
    return 0;
}

int launch_lattice_front(const KParams &p, cudaStream_t st) { return lat_launch(p, false, st); }
int launch_lattice_list(const KParams &p, cudaStream_t st) { return lat_launch(p, true, st); }

}  // namespace rtgpu
