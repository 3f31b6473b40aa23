// nrrs_render.cu -- the render front-end of trace_frame's depth 1 on the GPU
// (first part): camera rays with the per-path jitter stream,
// closest hits through the reference's BVH, dispatch and the surface vertex
// fields that feed the RRS stage.
//
//   camera_kernel     Camera::generate_ray (scene.cpp:10-21) at (x + j0, y + j1),
//                     j = path_stream(seed, root key, 1, CameraJitter) (wavefront.cpp:253-268)
//   intersect_kernel  Bvh::intersect (geometry.cpp:139-171): stack traversal, near
//                     child first, intersect_aabb (:74-83), intersect_triangle (:46-70)
//   surface_kernel    dispatch (wavefront.cpp:125-138) + Scene::interaction /
//                     normalize_position / dir_to_spherical01 (scene.cpp:50-96, core.hpp:52-58)
//
// Every float operation is an explicit round-to-nearest intrinsic (no FMA
// contraction) and min / max keep std::min / std::max's argument order, so the
// rays and hits equal the CPU reference's bit for bit.
#include "nrrs_device.cuh"
#include "nrrs_internal.h"

#include <cuda_runtime.h>

namespace nrrs {

namespace {
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float dot3(const float a[3], const float b[3]) {
    return fa(fa(fm(a[0], b[0]), fm(a[1], b[1])), fm(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const float a[3], const float b[3], float r[3]) {
    const float x = fs(fm(a[1], b[2]), fm(a[2], b[1]));
    const float y = fs(fm(a[2], b[0]), fm(a[0], b[2]));
    const float z = fs(fm(a[0], b[1]), fm(a[1], b[0]));
    r[0] = x;
    r[1] = y;
    r[2] = z;
}
__device__ __forceinline__ float stdmin(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ float stdmax(float a, float b) { return a < b ? b : a; }
}  // namespace

__global__ void camera_kernel(RenderScene s, uint32_t width, uint32_t height, uint64_t mixed_seed, uint32_t frame,
                              float *o, float *d, uint64_t *keys) {
    const uint64_t n = (uint64_t)width * height;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = mix_bits(((uint64_t)frame << 32) | p);  // root_path_key (rng.hpp:74-76)
        // path_stream(seed, key, 1, CameraJitter): the constructor's two steps, then two outputs
        constexpr uint64_t kMul = 6364136223846793005ull;
        const uint64_t seq = mix_bits(key ^ mix_bits((1ull << 8) ^ 0x11ull));
        const uint64_t inc = (seq << 1u) | 1u;
        uint64_t state = inc + mixed_seed;
        state = state * kMul + inc;
        const float j0 = fm((float)(pcg_output(state) >> 8), 0x1p-24f);
        state = state * kMul + inc;
        const float j1 = fm((float)(pcg_output(state) >> 8), 0x1p-24f);
        const float u = __fdiv_rn(fa((float)(p % width), j0), (float)width);
        const float v = __fdiv_rn(fa((float)(p / width), j1), (float)height);
        const float px = fm(fm(fs(fm(2.0f, u), 1.0f), s.tan_half), s.aspect);
        const float py = fm(fs(1.0f, fm(2.0f, v)), s.tan_half);
        float dir[3];
        for (int a = 0; a < 3; ++a)
            dir[a] = fa(fa(s.cam_fwd[a], fm(px, s.cam_right[a])), fm(py, s.cam_up[a]));
        const float sq = dot3(dir, dir);
        if (sq > 0.0f) {
            const float nrm = __fsqrt_rn(sq);
            for (int a = 0; a < 3; ++a)
                dir[a] = __fdiv_rn(dir[a], nrm);
        }
        for (int a = 0; a < 3; ++a) {
            o[3 * p + a] = s.cam_pos[a];
            d[3 * p + a] = dir[a];
        }
        keys[p] = key;
    }
}

// intersect_triangle (geometry.cpp:46-70)
__device__ __forceinline__ bool tri_hit(const RenderScene &s, uint32_t tri, const float o[3], const float d[3],
                                        float t_max, float &t, float &u, float &v) {
    const uint32_t i0 = s.idx[3 * tri], i1 = s.idx[3 * tri + 1], i2 = s.idx[3 * tri + 2];
    const float p0[3] = {s.pos[3 * i0], s.pos[3 * i0 + 1], s.pos[3 * i0 + 2]};
    const float e1[3] = {fs(s.pos[3 * i1], p0[0]), fs(s.pos[3 * i1 + 1], p0[1]), fs(s.pos[3 * i1 + 2], p0[2])};
    const float e2[3] = {fs(s.pos[3 * i2], p0[0]), fs(s.pos[3 * i2 + 1], p0[1]), fs(s.pos[3 * i2 + 2], p0[2])};
    float pv[3], qv[3];
    cross3(d, e2, pv);
    const float det = dot3(e1, pv);
    if (fabsf(det) < 1e-12f)
        return false;
    const float inv_det = __fdiv_rn(1.0f, det);
    const float tv[3] = {fs(o[0], p0[0]), fs(o[1], p0[1]), fs(o[2], p0[2])};
    const float uu = fm(dot3(tv, pv), inv_det);
    if (uu < 0.0f || uu > 1.0f)
        return false;
    cross3(tv, e1, qv);
    const float vv = fm(dot3(d, qv), inv_det);
    if (vv < 0.0f || fa(uu, vv) > 1.0f)
        return false;
    const float tt = fm(dot3(e2, qv), inv_det);
    if (tt <= 1e-4f || tt >= t || tt >= t_max)  // kRayEps (core.hpp:21)
        return false;
    t = tt;
    u = uu;
    v = vv;
    return true;
}

__global__ void intersect_kernel(RenderScene s, const float *ro, const float *rd, const float *rtmax, uint64_t n,
                                 float *out_t, uint32_t *out_tri, float *out_u, float *out_v, uint32_t *err) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const float o[3] = {ro[3 * r], ro[3 * r + 1], ro[3 * r + 2]};
        const float d[3] = {rd[3 * r], rd[3 * r + 1], rd[3 * r + 2]};
        const float t_max = rtmax ? rtmax[r] : __int_as_float(0x7f800000);
        float t = __int_as_float(0x7f800000), u = 0.0f, v = 0.0f;
        uint32_t tri = 0xFFFFFFFFu;
        // "Bvh::intersect: degenerate ray direction" (geometry.cpp:145-146): flagged, returned as a miss
        const bool degenerate = dot3(d, d) == 0.0f || !(isfinite(d[0]) && isfinite(d[1]) && isfinite(d[2]));
        if (degenerate)
            atomicOr(err, 1u);
        if (s.n_nodes > 0 && !degenerate) {
            const float inv_d[3] = {__fdiv_rn(1.0f, d[0]), __fdiv_rn(1.0f, d[1]), __fdiv_rn(1.0f, d[2])};
            uint32_t stack[64];
            int sp = 0;
            stack[sp++] = 0;
            while (sp > 0) {
                const uint32_t ni = stack[--sp];
                const BvhNodeDev node = s.nodes[ni];
                // intersect_aabb(node.bounds, o, inv_d, min(hit.t, t_max))
                float t0 = 0.0f, t1 = stdmin(t, t_max);
                for (int a = 0; a < 3; ++a) {
                    const float lo = fm(fs(node.lo[a], o[a]), inv_d[a]);
                    const float hi = fm(fs(node.hi[a], o[a]), inv_d[a]);
                    t0 = stdmax(t0, stdmin(lo, hi));
                    t1 = stdmin(t1, stdmax(lo, hi));
                }
                if (!(t0 <= t1))
                    continue;
                if (node.count > 0) {
                    for (uint32_t i = 0; i < node.count; ++i) {
                        const uint32_t prim = s.prims[node.offset + i];
                        if (tri_hit(s, prim, o, d, t_max, t, u, v))
                            tri = prim;
                    }
                } else {
                    const uint32_t left = ni + 1, right = node.offset;
                    if (inv_d[node.axis] >= 0.0f) {  // near child first by the split axis direction
                        stack[sp++] = right;
                        stack[sp++] = left;
                    } else {
                        stack[sp++] = left;
                        stack[sp++] = right;
                    }
                }
            }
        }
        out_t[r] = t;
        out_tri[r] = tri;
        if (out_u)
            out_u[r] = u;
        if (out_v)
            out_v[r] = v;
    }
}

// dispatch + the surface vertex fields of one hit (wavefront.cpp:125-138, :330-345)
__global__ void surface_kernel(RenderScene s, const float *ro, const float *rd, const float *hit_t,
                               const uint32_t *hit_tri, uint64_t n, uint8_t *cls, float *p01, float *wo01,
                               float *roughness, uint32_t *material) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t tri = hit_tri[r];
        uint8_t c = 0;
        float q[3] = {0.0f, 0.0f, 0.0f}, w2[2] = {0.0f, 0.0f}, rough = 0.0f;
        uint32_t m = 0xFFFFFFFFu;
        if (tri != 0xFFFFFFFFu) {
            m = s.mat_of_tri[tri];
            const float *alb = s.mat_albedo + 3 * m;
            const float amax = stdmax(stdmax(alb[0], alb[1]), alb[2]);
            const bool scattering = s.mat_kind[m] == 1 || amax > 0.0f;
            c = scattering ? 2 : 1;
            if (scattering) {
                const float t = hit_t[r];
                for (int a = 0; a < 3; ++a) {
                    const float pt = fa(ro[3 * r + a], fm(t, rd[3 * r + a]));
                    const float qq = fm(fs(pt, s.norm_offset[a]), s.norm_scale);
                    q[a] = stdmin(stdmax(qq, 0.0f), 1.0f);  // cwiseMax(0).cwiseMin(1)
                }
                const float wz = -rd[3 * r + 2];
                const float theta = acosf(wz < -1.0f ? -1.0f : (wz > 1.0f ? 1.0f : wz));
                float phi = atan2f(-rd[3 * r + 1], -rd[3 * r]);
                if (phi < 0.0f)
                    phi = fa(phi, fm(2.0f, 3.14159265358979323846f));
                w2[0] = fm(theta, 0.31830988618379067154f);
                w2[1] = fm(phi, fm(0.5f, 0.31830988618379067154f));
                rough = s.mat_kind[m] == 1 ? s.mat_roughness[m] : 1.0f;
            }
        }
        cls[r] = c;
        for (int a = 0; a < 3; ++a)
            p01[3 * r + a] = q[a];
        wo01[2 * r] = w2[0];
        wo01[2 * r + 1] = w2[1];
        roughness[r] = rough;
        if (material)
            material[r] = m;
    }
}

static uint32_t grid_for(uint64_t n, int num_sms) {
    const uint64_t want = (n + 255) / 256, cap = (uint64_t)num_sms * 16;
    return (uint32_t)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_camera(const RenderScene &s, uint32_t width, uint32_t height, uint64_t mixed_seed, uint32_t frame,
                          float *o, float *d, uint64_t *keys, int num_sms, cudaStream_t stream) {
    camera_kernel<<<grid_for((uint64_t)width * height, num_sms), 256, 0, stream>>>(s, width, height, mixed_seed, frame,
                                                                                 o, d, keys);
    return cudaGetLastError();
}

cudaError_t launch_intersect(const RenderScene &s, const float *o, const float *d, const float *tmax, uint64_t n,
                             float *t, uint32_t *tri, float *u, float *v, uint32_t *err, int num_sms,
                             cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    intersect_kernel<<<grid_for(n, num_sms), 256, 0, stream>>>(s, o, d, tmax, n, t, tri, u, v, err);
    return cudaGetLastError();
}

cudaError_t launch_surface(const RenderScene &s, const float *o, const float *d, const float *t, const uint32_t *tri,
                           uint64_t n, uint8_t *cls, float *p01, float *wo01, float *rough, uint32_t *material,
                           int num_sms, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    surface_kernel<<<grid_for(n, num_sms), 256, 0, stream>>>(s, o, d, t, tri, n, cls, p01, wo01, rough, material);
    return cudaGetLastError();
}

}  // namespace nrrs
