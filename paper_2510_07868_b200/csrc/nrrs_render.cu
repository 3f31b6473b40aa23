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

// path_stream(seed, key, depth, purpose): the constructor's two steps, then two outputs (rng.hpp:37-82)
__device__ __forceinline__ void path_floats2(uint64_t mixed_seed, uint64_t key, uint32_t depth, uint64_t purpose,
                                             float &a, float &b) {
    constexpr uint64_t kMul = 6364136223846793005ull;
    const uint64_t seq = mix_bits(key ^ mix_bits(((uint64_t)depth << 8) ^ purpose));
    const uint64_t inc = (seq << 1u) | 1u;
    uint64_t state = inc + mixed_seed;
    state = state * kMul + inc;
    a = fm((float)(pcg_output(state) >> 8), 0x1p-24f);
    state = state * kMul + inc;
    b = fm((float)(pcg_output(state) >> 8), 0x1p-24f);
}

// Camera::generate_ray at the jittered film position of pixel p (wavefront.cpp:253-268)
__device__ __forceinline__ uint64_t camera_ray(const RenderScene &s, uint32_t width, uint32_t height,
                                               uint64_t mixed_seed, uint32_t frame, uint64_t p, float dir[3]) {
    const uint64_t key = mix_bits(((uint64_t)frame << 32) | p);  // root_path_key (rng.hpp:74-76)
    float j0, j1;
    path_floats2(mixed_seed, key, 1, 0x11, j0, j1);  // Draw::CameraJitter
    const float u = __fdiv_rn(fa((float)(p % width), j0), (float)width);
    const float v = __fdiv_rn(fa((float)(p / width), j1), (float)height);
    const float px = fm(fm(fs(fm(2.0f, u), 1.0f), s.tan_half), s.aspect);
    const float py = fm(fs(1.0f, fm(2.0f, v)), s.tan_half);
    for (int a = 0; a < 3; ++a)
        dir[a] = fa(fa(s.cam_fwd[a], fm(px, s.cam_right[a])), fm(py, s.cam_up[a]));
    const float sq = dot3(dir, dir);
    if (sq > 0.0f) {
        const float nrm = __fsqrt_rn(sq);
        for (int a = 0; a < 3; ++a)
            dir[a] = __fdiv_rn(dir[a], nrm);
    }
    return key;
}

__global__ void camera_kernel(RenderScene s, uint32_t width, uint32_t height, uint64_t mixed_seed, uint32_t frame,
                              float *o, float *d, uint64_t *keys) {
    const uint64_t n = (uint64_t)width * height;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
        float dir[3];
        const uint64_t key = camera_ray(s, width, height, mixed_seed, frame, p, dir);
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

// intersect_triangle on the pre-gathered record of BVH prim slot k (p0, e1, e2 as the reference computes them)
__device__ __forceinline__ bool tri_hit_slot(const RenderScene &s, uint32_t k, const float o[3], const float d[3],
                                             float t_max, float &t, float &u, float &v, uint32_t &tri) {
    // generic loads: s.tri4 may point into shared memory (stage_scene)
    const float4 a = s.tri4[3 * (uint64_t)k], b = s.tri4[3 * (uint64_t)k + 1], c = s.tri4[3 * (uint64_t)k + 2];
    const float p0[3] = {a.x, a.y, a.z}, e1[3] = {a.w, b.x, b.y}, e2[3] = {b.z, b.w, c.x};
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
    tri = __float_as_uint(c.y);
    return true;
}

// Bvh::intersect (geometry.cpp:144-176); returns false for a degenerate direction (the reference throws)
__device__ __forceinline__ bool closest_hit(const RenderScene &s, const float o[3], const float d[3], float t_max,
                                            float &t, uint32_t &tri, float &u, float &v) {
    t = __int_as_float(0x7f800000);
    u = 0.0f;
    v = 0.0f;
    tri = 0xFFFFFFFFu;
    if (dot3(d, d) == 0.0f || !(isfinite(d[0]) && isfinite(d[1]) && isfinite(d[2])))
        return false;
    if (s.n_nodes == 0)
        return true;
    const float inv_d[3] = {__fdiv_rn(1.0f, d[0]), __fdiv_rn(1.0f, d[1]), __fdiv_rn(1.0f, d[2])};
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
#ifdef NRRS_WHILE_WHILE
    // while-while traversal: inner nodes until a leaf is reached, then the leaf.  Each ray visits
    // nodes and leaves in exactly the reference's order (a leaf is tested as soon as it is popped).
    while (sp > 0) {
        uint32_t leaf = 0xFFFFFFFFu;
        BvhNodeDev ln;
        while (sp > 0) {
            const uint32_t ni = stack[--sp];
            const BvhNodeDev node = s.nodes[ni];
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
                leaf = ni;
                ln = node;
                break;
            }
            const uint32_t left = ni + 1, right = node.offset;
            if (inv_d[node.axis] >= 0.0f) {
                stack[sp++] = right;
                stack[sp++] = left;
            } else {
                stack[sp++] = left;
                stack[sp++] = right;
            }
        }
        if (leaf != 0xFFFFFFFFu)
            for (uint32_t i = 0; i < ln.count; ++i) {
                const uint32_t prim = s.prims[ln.offset + i];
                if (tri_hit(s, prim, o, d, t_max, t, u, v))
                    tri = prim;
            }
    }
#else
    while (sp > 0) {
        const uint32_t ni = stack[--sp];
        const BvhNodeDev node = s.nodes[ni];
        // intersect_aabb(node.bounds, o, inv_d, min(hit.t, t_max)) (geometry.cpp:73-82)
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
            for (uint32_t i = 0; i < node.count; ++i)
                tri_hit_slot(s, node.offset + i, o, d, t_max, t, u, v, tri);
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
#endif
    return true;
}

// Bvh::occluded (geometry.cpp:178-202): any triangle hit in (kRayEps, t_max)
__device__ __forceinline__ bool any_hit(const RenderScene &s, const float o[3], const float d[3], float t_max) {
    if (s.n_nodes == 0)
        return false;
    const float inv_d[3] = {__fdiv_rn(1.0f, d[0]), __fdiv_rn(1.0f, d[1]), __fdiv_rn(1.0f, d[2])};
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const uint32_t ni = stack[--sp];
        const BvhNodeDev node = s.nodes[ni];
        float t0 = 0.0f, t1 = t_max;
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
                float t = t_max, u, v;
                uint32_t tr;
                if (tri_hit_slot(s, node.offset + i, o, d, t_max, t, u, v, tr))
                    return true;
            }
        } else {
            stack[sp++] = node.offset;
            stack[sp++] = ni + 1;
        }
    }
    return false;
}

__global__ void intersect_kernel(RenderScene s, const float *ro, const float *rd, const float *rtmax, uint64_t n,
                                 float *out_t, uint32_t *out_tri, float *out_u, float *out_v, uint32_t *err) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const float o[3] = {ro[3 * r], ro[3 * r + 1], ro[3 * r + 2]};
        const float d[3] = {rd[3 * r], rd[3 * r + 1], rd[3 * r + 2]};
        const float t_max = rtmax ? rtmax[r] : __int_as_float(0x7f800000);
        float t, u, v;
        uint32_t tri;
        // "Bvh::intersect: degenerate ray direction" (geometry.cpp:145-146): flagged, returned as a miss
        if (!closest_hit(s, o, d, t_max, t, tri, u, v))
            atomicOr(err, 1u);
        out_t[r] = t;
        out_tri[r] = tri;
        if (out_u)
            out_u[r] = u;
        if (out_v)
            out_v[r] = v;
    }
}

// dir_to_spherical01 (core.hpp:52-58).  acos / atan2 are evaluated in double and rounded once,
// i.e. correctly rounded like glibc's acosf / atan2f in all but rare halfway cases.
__device__ __forceinline__ void spherical01(const float wo[3], float out[2]) {
    const float z = wo[2] < -1.0f ? -1.0f : (wo[2] > 1.0f ? 1.0f : wo[2]);
    const float theta = __double2float_rn(acos((double)z));
    float phi = __double2float_rn(atan2((double)wo[1], (double)wo[0]));
    if (phi < 0.0f)
        phi = fa(phi, fm(2.0f, 3.14159265358979323846f));
    out[0] = fm(theta, 0.31830988618379067154f);
    out[1] = fm(phi, fm(0.5f, 0.31830988618379067154f));
}

// Scene::normalize_position (scene.cpp:93-96)
__device__ __forceinline__ void normalize_position(const RenderScene &s, const float p[3], float q[3]) {
    for (int a = 0; a < 3; ++a) {
        const float qq = fm(fs(p[a], s.norm_offset[a]), s.norm_scale);
        q[a] = stdmin(stdmax(qq, 0.0f), 1.0f);  // cwiseMax(0).cwiseMin(1)
    }
}

// TriMesh::face_normal (geometry.cpp:22-28)
__device__ __forceinline__ void face_normal(const RenderScene &s, uint32_t tri, float n[3]) {
    const uint32_t i0 = s.idx[3 * tri], i1 = s.idx[3 * tri + 1], i2 = s.idx[3 * tri + 2];
    const float e1[3] = {fs(s.pos[3 * i1], s.pos[3 * i0]), fs(s.pos[3 * i1 + 1], s.pos[3 * i0 + 1]),
                         fs(s.pos[3 * i1 + 2], s.pos[3 * i0 + 2])};
    const float e2[3] = {fs(s.pos[3 * i2], s.pos[3 * i0]), fs(s.pos[3 * i2 + 1], s.pos[3 * i0 + 1]),
                         fs(s.pos[3 * i2 + 2], s.pos[3 * i0 + 2])};
    float c[3];
    cross3(e1, e2, c);
    const float len = __fsqrt_rn(dot3(c, c));
    if (len > 0.0f) {
        for (int a = 0; a < 3; ++a)
            n[a] = __fdiv_rn(c[a], len);
    } else {
        n[0] = 0.0f;
        n[1] = 0.0f;
        n[2] = 1.0f;
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
                float pt[3];
                for (int a = 0; a < 3; ++a)
                    pt[a] = fa(ro[3 * r + a], fm(t, rd[3 * r + a]));
                normalize_position(s, pt, q);
                const float wo[3] = {-rd[3 * r], -rd[3 * r + 1], -rd[3 * r + 2]};
                spherical01(wo, w2);
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

// ============================================================================
// trace_frame on the GPU: shade, vertex records, scatter
// (NEE + BSDF sampling per child slot) and the ordered film / parent folds.
// ============================================================================
constexpr float kPiF = 3.14159265358979323846f;
constexpr float kInvPiF = 0.31830988618379067154f;

__device__ __forceinline__ float max3(const float v[3]) { return stdmax(stdmax(v[0], v[1]), v[2]); }  // maxCoeff
__device__ __forceinline__ float fdv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fsq(float a) { return __fsqrt_rn(a); }

// mis_power2 (wavefront.cpp:15-21), squares in double
__device__ __forceinline__ float mis_power2(float a, float b) {
    const double a2 = __dmul_rn((double)a, (double)a), b2 = __dmul_rn((double)b, (double)b);
    const double sum = __dadd_rn(a2, b2);
    if (sum <= 0.0)
        return 0.0f;
    return __double2float_rn(__ddiv_rn(a2, sum));
}

// build_frame (core.hpp:43-50) + to_world (bsdf.cpp:35-39)
__device__ __forceinline__ void to_world(const float n[3], const float l[3], float w[3]) {
    const float sign = copysignf(1.0f, n[2]);
    const float a = fdv(-1.0f, fa(sign, n[2]));
    const float c = fm(fm(n[0], n[1]), a);
    const float t[3] = {fa(1.0f, fm(fm(fm(sign, n[0]), n[0]), a)), fm(sign, c), fm(-sign, n[0])};
    const float b[3] = {c, fa(sign, fm(fm(n[1], n[1]), a)), -n[1]};
    for (int k = 0; k < 3; ++k)
        w[k] = fa(fa(fm(l[0], t[k]), fm(l[1], b[k])), fm(l[2], n[k]));
}

// bsdf.cpp:14-33
__device__ __forceinline__ float ggx_d(float cos_h, float alpha) {
    if (cos_h <= 0.0f)
        return 0.0f;
    const float a2 = fm(alpha, alpha);
    const float d = stdmax(fa(fm(fm(cos_h, cos_h), fs(a2, 1.0f)), 1.0f), 1e-12f);
    return fdv(a2, fm(fm(kPiF, d), d));
}
__device__ __forceinline__ float smith_g1(float cos_v, float alpha) {
    if (cos_v <= 0.0f)
        return 0.0f;
    const float a2 = fm(alpha, alpha);
    return fdv(fm(2.0f, cos_v), fa(cos_v, fsq(fa(a2, fm(fm(fs(1.0f, a2), cos_v), cos_v)))));
}
__device__ __forceinline__ void schlick(const float f0[3], float cos_i, float out[3]) {
    float m = fs(1.0f, cos_i);
    m = m < 0.0f ? 0.0f : (1.0f < m ? 1.0f : m);  // std::clamp
    const float m2 = fm(m, m);
    const float w = fm(fm(m2, m2), m);
    for (int a = 0; a < 3; ++a)
        out[a] = fa(f0[a], fm(fs(1.0f, f0[a]), w));
}
__device__ __forceinline__ void half_vec(const float wo[3], const float wi[3], float h[3]) {
    for (int a = 0; a < 3; ++a)
        h[a] = fa(wo[a], wi[a]);
    const float sq = dot3(h, h);
    if (sq > 0.0f) {
        const float nn = fsq(sq);
        for (int a = 0; a < 3; ++a)
            h[a] = fdv(h[a], nn);
    }
}

struct MatView {
    int kind;
    float alb[3], rough;
};

// bsdf_eval (bsdf.cpp:43-61)
__device__ __forceinline__ void bsdf_eval(const MatView &m, const float n[3], const float wo[3], const float wi[3],
                                          float f[3]) {
    f[0] = f[1] = f[2] = 0.0f;
    const float cos_o = dot3(n, wo), cos_i = dot3(n, wi);
    if (cos_o <= 0.0f || cos_i <= 0.0f)
        return;
    if (m.kind == 0) {
        for (int a = 0; a < 3; ++a)
            f[a] = fm(m.alb[a], kInvPiF);
        return;
    }
    float h[3], fr[3];
    half_vec(wo, wi, h);
    const float alpha = stdmax(m.rough, 1e-3f);
    const float d = ggx_d(dot3(n, h), alpha);
    const float g = fm(smith_g1(cos_o, alpha), smith_g1(cos_i, alpha));
    schlick(m.alb, dot3(wo, h), fr);
    const float sc = fdv(fm(d, g), fm(fm(4.0f, cos_o), cos_i));
    for (int a = 0; a < 3; ++a)
        f[a] = fm(fr[a], sc);
}
// bsdf_pdf (bsdf.cpp:63-83)
__device__ __forceinline__ float bsdf_pdf(const MatView &m, const float n[3], const float wo[3], const float wi[3]) {
    const float cos_o = dot3(n, wo), cos_i = dot3(n, wi);
    if (cos_o <= 0.0f || cos_i <= 0.0f)
        return 0.0f;
    if (m.kind == 0)
        return fm(cos_i, kInvPiF);
    float h[3];
    half_vec(wo, wi, h);
    const float cos_h = dot3(n, h);
    const float d = ggx_d(cos_h, stdmax(m.rough, 1e-3f));
    const float dot_oh = dot3(wo, h);
    if (dot_oh <= 0.0f)
        return 0.0f;
    return fdv(fm(d, cos_h), fm(4.0f, dot_oh));
}
// std::cos / std::sin of a float: evaluated in double, rounded once
__device__ __forceinline__ float cos_rn(float x) { return __double2float_rn(cos((double)x)); }
__device__ __forceinline__ float sin_rn(float x) { return __double2float_rn(sin((double)x)); }

// bsdf_sample (bsdf.cpp:85-133)
__device__ __forceinline__ bool bsdf_sample(const MatView &m, const float n[3], const float wo[3], float u1,
                                            float u2, float wi[3], float &pdf, float thr[3]) {
    const float cos_o = dot3(n, wo);
    if (cos_o <= 0.0f)
        return false;
    if (m.kind == 0) {
        const float r = fsq(u1);
        const float phi = fm(fm(2.0f, kPiF), u2);
        const float loc[3] = {fm(r, cos_rn(phi)), fm(r, sin_rn(phi)), fsq(stdmax(0.0f, fs(1.0f, u1)))};
        to_world(n, loc, wi);
        const float cos_i = dot3(n, wi);
        if (cos_i <= 0.0f)
            return false;
        pdf = fm(cos_i, kInvPiF);
        thr[0] = m.alb[0];
        thr[1] = m.alb[1];
        thr[2] = m.alb[2];
        return true;
    }
    const float alpha = stdmax(m.rough, 1e-3f);
    const float tan2 = fdv(fm(fm(alpha, alpha), u1), stdmax(fs(1.0f, u1), 1e-12f));
    const float cos_h = fdv(1.0f, fsq(fa(1.0f, tan2)));
    const float sin_h = fsq(stdmax(0.0f, fs(1.0f, fm(cos_h, cos_h))));
    const float phi = fm(fm(2.0f, kPiF), u2);
    const float loc[3] = {fm(sin_h, cos_rn(phi)), fm(sin_h, sin_rn(phi)), cos_h};
    float h[3], fr[3];
    to_world(n, loc, h);
    const float dot_oh = dot3(wo, h);
    if (dot_oh <= 0.0f)
        return false;
    for (int a = 0; a < 3; ++a)
        wi[a] = fs(fm(fm(2.0f, dot_oh), h[a]), wo[a]);
    const float cos_i = dot3(n, wi);
    if (cos_i <= 0.0f)
        return false;
    const float nh = dot3(n, h);
    pdf = fdv(fm(ggx_d(nh, alpha), nh), fm(4.0f, dot_oh));
    if (!(pdf > 0.0f) || !isfinite(pdf))
        return false;
    const float g = fm(smith_g1(cos_o, alpha), smith_g1(cos_i, alpha));
    schlick(m.alb, dot_oh, fr);
    const float sc = fdv(fm(g, dot_oh), fm(cos_o, nh));
    for (int a = 0; a < 3; ++a)
        thr[a] = fm(fr[a], sc);
    return true;
}

__device__ __forceinline__ MatView mat_view(const RenderScene &s, uint32_t m) {
    MatView v;
    v.kind = s.mat_kind[m];
    v.alb[0] = s.mat_albedo[3 * m];
    v.alb[1] = s.mat_albedo[3 * m + 1];
    v.alb[2] = s.mat_albedo[3 * m + 2];
    v.rough = s.mat_roughness[m];
    return v;
}

// hit_emission (wavefront.cpp:28-41)
__device__ __forceinline__ void hit_emission(const RenderScene &s, const float d[3], uint32_t tri, float dist,
                                             float prev_pdf, float out[3]) {
    const uint32_t m = s.mat_of_tri[tri];
    const float e[3] = {s.mat_emission[3 * m], s.mat_emission[3 * m + 1], s.mat_emission[3 * m + 2]};
    out[0] = out[1] = out[2] = 0.0f;
    if (!(max3(e) > 0.0f))
        return;
    float mis = 1.0f;
    if (prev_pdf >= 0.0f) {
        const int32_t li = s.light_index[tri];
        const float pdf_area = li < 0 ? 0.0f : fdv(1.0f, fm((float)s.n_lights, s.light_areas[li]));
        if (pdf_area > 0.0f) {
            float nl[3];
            face_normal(s, tri, nl);
            const float cos_l = fabsf(dot3(nl, d));
            const float pdf_sa = fdv(fm(fm(pdf_area, dist), dist), stdmax(cos_l, 1e-8f));
            mis = mis_power2(prev_pdf, pdf_sa);
        }
    }
    for (int a = 0; a < 3; ++a)
        out[a] = fm(e[a], mis);
}

// BVH nodes and triangle records staged into this CTA's shared memory when the launch gave room
// for them (scene_smem_bytes): the walks' dependent node / triangle loads then hit smem instead of
// L1/L2.  Same data, same arithmetic.  All threads of the CTA must call it.
__device__ __forceinline__ RenderScene stage_scene(const RenderScene &s) {
    extern __shared__ __align__(16) uint8_t scene_smem[];
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    RenderScene ls = s;
    const uint32_t nb = s.n_nodes * (uint32_t)sizeof(BvhNodeDev), tb = s.n_tri * 48u;
    if (dyn != 0 && dyn >= nb + tb) {
        const uint4 *sn = reinterpret_cast<const uint4 *>(s.nodes), *st4 = reinterpret_cast<const uint4 *>(s.tri4);
        uint4 *dn = reinterpret_cast<uint4 *>(scene_smem), *dt = reinterpret_cast<uint4 *>(scene_smem + nb);
        for (uint32_t i = threadIdx.x; i < nb / 16u; i += blockDim.x)
            dn[i] = __ldg(sn + i);
        for (uint32_t i = threadIdx.x; i < tb / 16u; i += blockDim.x)
            dt[i] = __ldg(st4 + i);
        ls.nodes = reinterpret_cast<const BvhNodeDev *>(scene_smem);
        ls.tri4 = reinterpret_cast<const float4 *>(scene_smem + nb);
    }
    __syncthreads();
    return ls;
}

// Per queue entry: closest hit, dispatch class (0 miss, 1 light, 2 surface), the miss / light
// film term (f64, zero when the reference adds nothing), depth-1 light normals, and the
// (entry, triangle) pair the surface compaction keeps.
__global__ void trace_shade_kernel(RenderScene s_in, const PathStateDev *q, uint32_t n, uint32_t depth, uint8_t *cls,
                                   uint8_t *is_surf, float *hit_t, uint32_t *pair, double *term, float *normals,
                                   uint32_t *err) {
    const RenderScene s = stage_scene(s_in);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const PathStateDev &st = q[i];
        const float o[3] = {st.o[0], st.o[1], st.o[2]}, d[3] = {st.d[0], st.d[1], st.d[2]};
        float t, u, v;
        uint32_t tri;
        if (!closest_hit(s, o, d, st.t_max, t, tri, u, v))
            atomicOr(err, 1u);
        uint8_t c = 0;
        double tm[3] = {0.0, 0.0, 0.0};
        if (tri == 0xFFFFFFFFu) {
            if (max3(s.env) > 0.0f)
                for (int a = 0; a < 3; ++a)
                    tm[a] = (double)fm(st.w[a], s.env[a]);
        } else {
            const uint32_t m = s.mat_of_tri[tri];
            const float *alb = s.mat_albedo + 3 * m;
            c = (s.mat_kind[m] == 1 || stdmax(stdmax(alb[0], alb[1]), alb[2]) > 0.0f) ? 2 : 1;
            if (c == 1) {
                if (depth == 1 && normals) {
                    float nl[3];
                    face_normal(s, tri, nl);
                    if (dot3(nl, d) > 0.0f)
                        for (int a = 0; a < 3; ++a)
                            nl[a] = -nl[a];
                    for (int a = 0; a < 3; ++a)
                        normals[3 * (uint64_t)st.pixel + a] = nl[a];
                }
                float em[3];
                hit_emission(s, d, tri, t, st.prev_pdf, em);
                if (max3(em) > 0.0f)
                    for (int a = 0; a < 3; ++a)
                        tm[a] = (double)fm(st.w[a], em[a]);
            }
        }
        cls[i] = c;
        is_surf[i] = c == 2;
        hit_t[i] = t;
        pair[2 * (uint64_t)i] = i;
        pair[2 * (uint64_t)i + 1] = tri;
        for (int a = 0; a < 3; ++a)
            term[3 * (uint64_t)i + a] = tm[a];
    }
}

// Surface vertex j = the j-th surface entry (wavefront.cpp:324-352); s starts as the emission term.
__global__ void trace_records_kernel(RenderScene s, const PathStateDev *q, const uint32_t *surf, const uint32_t *ns_p,
                                     uint32_t n_max, const float *hit_t, uint32_t *rank, VertexRecDev v,
                                     uint32_t depth, float *normals) {
    const uint32_t ns = *ns_p < n_max ? *ns_p : n_max;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < ns; j += gridDim.x * blockDim.x) {
        const uint32_t i = surf[2 * (uint64_t)j], tri = surf[2 * (uint64_t)j + 1];
        rank[i] = j;
        const PathStateDev &st = q[i];
        const float d[3] = {st.d[0], st.d[1], st.d[2]};
        const float t = hit_t[i];
        float p[3], wo[3], n[3], q01[3], w2[2];
        for (int a = 0; a < 3; ++a) {
            p[a] = fa(st.o[a], fm(t, d[a]));
            wo[a] = -d[a];
        }
        face_normal(s, tri, n);  // shading_normal without per-vertex normals (geometry.cpp:30-38)
        if (dot3(n, wo) < 0.0f)
            for (int a = 0; a < 3; ++a)
                n[a] = -n[a];
        normalize_position(s, p, q01);
        spherical01(wo, w2);
        const uint32_t m = s.mat_of_tri[tri];
        float em[3];
        hit_emission(s, d, tri, t, st.prev_pdf, em);
        const bool emits = max3(em) > 0.0f;
        for (int a = 0; a < 3; ++a) {
            v.p[3 * (uint64_t)j + a] = p[a];
            v.n_s[3 * (uint64_t)j + a] = n[a];
            v.wo[3 * (uint64_t)j + a] = wo[a];
            v.weight[3 * (uint64_t)j + a] = st.w[a];
            v.p01[3 * (uint64_t)j + a] = q01[a];
            v.s[3 * (uint64_t)j + a] = emits ? (double)fm(st.w[a], em[a]) : 0.0;
        }
        v.wo01[2 * (uint64_t)j] = w2[0];
        v.wo01[2 * (uint64_t)j + 1] = w2[1];
        v.rough[j] = s.mat_kind[m] == 1 ? s.mat_roughness[m] : 1.0f;
        v.material[j] = m;
        v.pixel[j] = st.pixel;
        v.parent[j] = st.parent;
        v.key[j] = st.key;
        v.rrs[j] = st.rrs;
        v.q_norm[j] = 1.0f;
        v.q_real[j] = 1.0f;
        v.decided[j] = 0;
        if (depth == 1 && normals)
            for (int a = 0; a < 3; ++a)
                normals[3 * (uint64_t)st.pixel + a] = n[a];
    }
}

// One child slot (wavefront.cpp:418-482): NEE term of the slot (f64, folded per vertex in child
// order later) and the child PathState; slot_used marks sampled children.
#ifndef NRRS_SCATTER_MINB
#define NRRS_SCATTER_MINB 4  // 64 registers: occupancy over the divergent walks (measured -5% frame time)
#endif
__global__ void __launch_bounds__(256, NRRS_SCATTER_MINB) trace_scatter_kernel(RenderScene s_in, VertexRecDev v, const uint32_t *slots, uint32_t spawned,
                                     uint32_t depth, uint64_t mixed_seed, PathStateDev *next, uint8_t *used,
                                     double *slot_term, TraceCounters *cnt) {
    const RenderScene s = stage_scene(s_in);
    uint32_t shadows = 0, nonfinite = 0;
    for (uint32_t sl = blockIdx.x * blockDim.x + threadIdx.x; sl < spawned; sl += gridDim.x * blockDim.x) {
        const uint32_t j = slots[2 * (uint64_t)sl], c = slots[2 * (uint64_t)sl + 1];
        const float p[3] = {v.p[3 * (uint64_t)j], v.p[3 * (uint64_t)j + 1], v.p[3 * (uint64_t)j + 2]};
        const float n[3] = {v.n_s[3 * (uint64_t)j], v.n_s[3 * (uint64_t)j + 1], v.n_s[3 * (uint64_t)j + 2]};
        const float wo[3] = {v.wo[3 * (uint64_t)j], v.wo[3 * (uint64_t)j + 1], v.wo[3 * (uint64_t)j + 2]};
        const float w[3] = {v.weight[3 * (uint64_t)j], v.weight[3 * (uint64_t)j + 1], v.weight[3 * (uint64_t)j + 2]};
        const MatView m = mat_view(s, v.material[j]);
        const float qr = v.q_real[j];
        const uint64_t ck = mix_bits(v.key[j] ^ mix_bits(0xc2b2ae3d27d4eb4full + c));  // child_path_key
        double nee[3] = {0.0, 0.0, 0.0};
        float pick, dummy, l1, l2;
        path_floats2(mixed_seed, ck, depth, 0x33, pick, dummy);  // Draw::LightPick
        path_floats2(mixed_seed, ck, depth, 0x44, l1, l2);       // Draw::LightPoint
        if (s.n_lights > 0) {  // sample_nee (wavefront.cpp:155-184), Scene::sample_light (scene.cpp:66-82)
            uint32_t li = (uint32_t)fm(pick, (float)s.n_lights);
            li = li < s.n_lights - 1 ? li : s.n_lights - 1;
            const uint32_t lt = s.light_tris[li];
            const float su = fsq(l1);
            const float bu = fs(1.0f, su), bv = fm(l2, su);
            const uint32_t i0 = s.idx[3 * lt], i1 = s.idx[3 * lt + 1], i2 = s.idx[3 * lt + 2];
            float lp[3], ln[3], wl[3];
            const float bw = fs(fs(1.0f, bu), bv);
            for (int a = 0; a < 3; ++a)
                lp[a] = fa(fa(fm(bw, s.pos[3 * i0 + a]), fm(bu, s.pos[3 * i1 + a])), fm(bv, s.pos[3 * i2 + a]));
            face_normal(s, lt, ln);
            const uint32_t lm = s.mat_of_tri[lt];
            const float le[3] = {s.mat_emission[3 * lm], s.mat_emission[3 * lm + 1], s.mat_emission[3 * lm + 2]};
            const float pdf_area = fdv(1.0f, fm((float)s.n_lights, s.light_areas[li]));
            if (pdf_area > 0.0f) {
                for (int a = 0; a < 3; ++a)
                    wl[a] = fs(lp[a], p[a]);
                const float dist2 = dot3(wl, wl);
                if (dist2 > 1e-12f) {
                    const float dist = fsq(dist2);
                    for (int a = 0; a < 3; ++a)
                        wl[a] = fdv(wl[a], dist);
                    const float cos_l = fabsf(dot3(ln, wl));
                    if (cos_l > 1e-7f) {
                        float f[3];
                        bsdf_eval(m, n, wo, wl, f);
                        const float cos_v = dot3(n, wl);
                        if (!(cos_v <= 0.0f || max3(f) <= 0.0f || max3(le) <= 0.0f)) {
                            const float scale = fdv(fm(cos_v, cos_l), fm(dist2, pdf_area));
                            const float pdf_l = fdv(fm(pdf_area, dist2), stdmax(cos_l, 1e-8f));
                            const float pdf_b = bsdf_pdf(m, n, wo, wl);
                            ++shadows;
                            if (!any_hit(s, p, wl, fm(dist, fs(1.0f, 1e-3f)))) {
                                const float mis = mis_power2(pdf_l, pdf_b);
                                for (int a = 0; a < 3; ++a)
                                    nee[a] = (double)fm(fdv(w[a], qr), fm(fm(fm(f[a], le[a]), scale), mis));
                            }
                        }
                    }
                }
            }
        }
        for (int a = 0; a < 3; ++a)
            slot_term[3 * (uint64_t)sl + a] = nee[a];
        float b1, b2, wi[3], pdf, thr[3];
        path_floats2(mixed_seed, ck, depth, 0x22, b1, b2);  // Draw::Bsdf
        uint8_t ok = 0;
        if (bsdf_sample(m, n, wo, b1, b2, wi, pdf, thr)) {
            PathStateDev ch;
            for (int a = 0; a < 3; ++a) {
                ch.o[a] = p[a];
                ch.d[a] = wi[a];
                ch.w[a] = fdv(fm(w[a], thr[a]), qr);
            }
            ch.t_max = __int_as_float(0x7f800000);
            if (!(isfinite(ch.w[0]) && isfinite(ch.w[1]) && isfinite(ch.w[2]))) {
                ++nonfinite;
            } else {
                ch.key = ck;
                ch.prev_pdf = pdf;
                ch.rrs = fm(v.rrs[j], qr);
                ch.pixel = v.pixel[j];
                ch.parent = (int32_t)j;
                ch.depth = (uint16_t)(depth + 1);
                ch.pad16 = 0;
                ch.pad = 0;
                next[sl] = ch;
                ok = 1;
            }
        }
        used[sl] = ok;
    }
    if (shadows)
        atomicAdd(&cnt->shadow_rays, (unsigned long long)shadows);
    if (nonfinite)
        atomicAdd(&cnt->nonfinite, (unsigned long long)nonfinite);
}

// frame[pixel] in the reference's order, one thread per pixel run of the queue:
// misses (:295-303), pure emitters (:305-321), surface emission (:353-356), NEE (:484-487);
// also s[j] += nee[j].  spawned == 0 / slot_term == NULL: terminal depth, no NEE.
__global__ void trace_fold_frame_kernel(const PathStateDev *q, uint32_t n, const uint8_t *cls, const double *term,
                                        const uint32_t *rank, VertexRecDev v, uint32_t spawned,
                                        const double *slot_term, double *frame) {
    const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 >= n)
        return;
    const uint32_t px = q[i0].pixel;
    if (i0 > 0 && q[i0 - 1].pixel == px)
        return;
    uint32_t end = i0 + 1;
    while (end < n && q[end].pixel == px)
        ++end;
    double f[3] = {frame[3 * (uint64_t)px], frame[3 * (uint64_t)px + 1], frame[3 * (uint64_t)px + 2]};
    for (int pass = 0; pass < 2; ++pass)
        for (uint32_t i = i0; i < end; ++i)
            if (cls[i] == pass)
                for (int a = 0; a < 3; ++a)
                    f[a] = __dadd_rn(f[a], term[3 * (uint64_t)i + a]);
    for (uint32_t i = i0; i < end; ++i)
        if (cls[i] == 2) {
            const uint32_t j = rank[i];
            for (int a = 0; a < 3; ++a)
                f[a] = __dadd_rn(f[a], v.s[3 * (uint64_t)j + a]);
        }
    if (slot_term)
        for (uint32_t i = i0; i < end; ++i)
            if (cls[i] == 2) {
                const uint32_t j = rank[i];
                const uint32_t off = v.offset[j];
                const uint32_t rem = spawned - (spawned < off ? spawned : off);
                const uint32_t kept = (uint32_t)v.k[j] < rem ? (uint32_t)v.k[j] : rem;
                double nee[3] = {0.0, 0.0, 0.0};
                for (uint32_t c = 0; c < kept; ++c)
                    for (int a = 0; a < 3; ++a)
                        nee[a] = __dadd_rn(nee[a], slot_term[3 * (uint64_t)(off + c) + a]);
                for (int a = 0; a < 3; ++a) {
                    f[a] = __dadd_rn(f[a], nee[a]);
                    v.s[3 * (uint64_t)j + a] = __dadd_rn(v.s[3 * (uint64_t)j + a], nee[a]);
                }
            }
    for (int a = 0; a < 3; ++a)
        frame[3 * (uint64_t)px + a] = f[a];
}

// (*up)[parent].s in the reference's order: misses, then pure emitters (:300-301, :318-319)
__global__ void trace_fold_parent_kernel(const PathStateDev *q, uint32_t n, const uint8_t *cls, const double *term,
                                         double *up_s) {
    const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 >= n)
        return;
    const int32_t par = q[i0].parent;
    if (i0 > 0 && q[i0 - 1].parent == par)
        return;
    if (par < 0)
        return;
    uint32_t end = i0 + 1;
    while (end < n && q[end].parent == par)
        ++end;
    double f[3] = {up_s[3 * (uint64_t)par], up_s[3 * (uint64_t)par + 1], up_s[3 * (uint64_t)par + 2]};
    for (int pass = 0; pass < 2; ++pass)
        for (uint32_t i = i0; i < end; ++i)
            if (cls[i] == pass)
                for (int a = 0; a < 3; ++a)
                    f[a] = __dadd_rn(f[a], term[3 * (uint64_t)i + a]);
    for (int a = 0; a < 3; ++a)
        up_s[3 * (uint64_t)par + a] = f[a];
}

__global__ void trace_camera_kernel(RenderScene s, uint32_t width, uint32_t height, uint64_t mixed_seed,
                                    uint32_t frame, PathStateDev *q) {
    const uint64_t n = (uint64_t)width * height;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
        PathStateDev st;
        st.key = camera_ray(s, width, height, mixed_seed, frame, p, st.d);
        for (int a = 0; a < 3; ++a) {
            st.o[a] = s.cam_pos[a];
            st.w[a] = 1.0f;
        }
        st.t_max = __int_as_float(0x7f800000);
        st.prev_pdf = -1.0f;
        st.rrs = 1.0f;
        st.pixel = (uint32_t)p;
        st.parent = -1;
        st.depth = 1;
        st.pad16 = 0;
        st.pad = 0;
        q[p] = st;
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

cudaError_t launch_trace_camera(const RenderScene &s, uint32_t width, uint32_t height, uint64_t mixed_seed,
                                uint32_t frame, PathStateDev *q, int num_sms, cudaStream_t stream) {
    trace_camera_kernel<<<grid_for((uint64_t)width * height, num_sms), 256, 0, stream>>>(s, width, height, mixed_seed,
                                                                                         frame, q);
    return cudaGetLastError();
}

// Dynamic smem for stage_scene: the scene's nodes + triangle records when they fit in 16 KB
// (a few CTAs per SM keep their occupancy), else 0 (walks read global memory).
static size_t scene_smem_bytes(const RenderScene &s) {
    const size_t b = (size_t)s.n_nodes * sizeof(BvhNodeDev) + (size_t)s.n_tri * 48u;
    return b <= 16384 ? b : 0;
}

cudaError_t launch_trace_shade(const RenderScene &s, const PathStateDev *q, uint32_t n, uint32_t depth,
                               uint8_t *cls, uint8_t *is_surf, float *hit_t, uint32_t *pair, double *term,
                               float *normals, uint32_t *err, int num_sms, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    trace_shade_kernel<<<grid_for(n, num_sms), 256, scene_smem_bytes(s), stream>>>(s, q, n, depth, cls, is_surf, hit_t, pair, term,
                                                                 normals, err);
    return cudaGetLastError();
}

cudaError_t launch_trace_records(const RenderScene &s, const PathStateDev *q, const uint32_t *surf, const uint32_t *ns,
                                 uint32_t n_max, const float *hit_t, uint32_t *rank, VertexRecDev v, uint32_t depth,
                                 float *normals, int num_sms, cudaStream_t stream) {
    if (n_max == 0)
        return cudaSuccess;
    trace_records_kernel<<<grid_for(n_max, num_sms), 256, 0, stream>>>(s, q, surf, ns, n_max, hit_t, rank, v, depth,
                                                                       normals);
    return cudaGetLastError();
}

cudaError_t launch_trace_scatter(const RenderScene &s, VertexRecDev v, const uint32_t *slots, uint32_t spawned,
                                 uint32_t depth, uint64_t mixed_seed, PathStateDev *next, uint8_t *used,
                                 double *slot_term, TraceCounters *cnt, int num_sms, cudaStream_t stream) {
    if (spawned == 0)
        return cudaSuccess;
    trace_scatter_kernel<<<grid_for(spawned, num_sms), 256, scene_smem_bytes(s), stream>>>(s, v, slots, spawned, depth, mixed_seed, next,
                                                                         used, slot_term, cnt);
    return cudaGetLastError();
}

cudaError_t launch_trace_fold_frame(const PathStateDev *q, uint32_t n, const uint8_t *cls, const double *term,
                                    const uint32_t *rank, VertexRecDev v, uint32_t spawned, const double *slot_term,
                                    double *frame, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    trace_fold_frame_kernel<<<(n + 255) / 256, 256, 0, stream>>>(q, n, cls, term, rank, v, spawned, slot_term, frame);
    return cudaGetLastError();
}

cudaError_t launch_trace_fold_parent(const PathStateDev *q, uint32_t n, const uint8_t *cls, const double *term,
                                     double *up_s, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    trace_fold_parent_kernel<<<(n + 255) / 256, 256, 0, stream>>>(q, n, cls, term, up_s);
    return cudaGetLastError();
}

}  // namespace nrrs
