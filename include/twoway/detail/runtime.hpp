#pragma once
// Header-only glue between the reference C++ API (include/twoway/*.hpp) and
// the C-ABI of libtwoway_b200.so (include/tw_c.h): one lazily created context
// per (host thread, device), topology uploads cached per (device, MeshState)
// and keyed by a topology hash, status -> exception mapping, and the
// Positions <-> N x 3 double conversions.
//
// Everything here is inline: it compiles against the caller's Vec3 (the
// header's own type or Eigen::Vector3d with TWOWAY_USE_EIGEN), so one prebuilt
// library serves both (the .so exports only extern "C" symbols).

#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tw_c.h"
#include "twoway/mesh.hpp"

namespace twoway::detail {

struct CtxDelete {
    void operator()(tw_ctx* c) const { tw_ctx_destroy(c); }
};
struct MeshDelete {
    void operator()(tw_mesh* m) const { tw_mesh_destroy(m); }
};
using CtxPtr = std::unique_ptr<tw_ctx, CtxDelete>;
using MeshPtr = std::unique_ptr<tw_mesh, MeshDelete>;

struct Runtime {
    struct Upload {
        uint64_t hash = 0;
        MeshPtr mesh;
    };
    std::map<int, CtxPtr> contexts;                              // by device
    std::map<std::pair<int, const MeshState*>, Upload> uploads;  // by (device, mesh)
    ~Runtime() {
        uploads.clear();  // meshes before their contexts
        contexts.clear();
    }
};

inline Runtime& runtime() {
    thread_local Runtime rt;
    return rt;
}

[[noreturn]] inline void raise_status(int rc, const tw_ctx* ctx) {
    const std::string msg = ctx ? tw_last_error(ctx) : "twoway: device call failed";
    if (rc == TW_EINVAL || rc == TW_EUNSUPPORTED) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void check(int rc, const tw_ctx* ctx) {
    if (rc != TW_OK) raise_status(rc, ctx);
}

inline tw_ctx* context(int device) {
    CtxPtr& slot = runtime().contexts[device];
    if (!slot) {
        tw_ctx* c = nullptr;
        if (tw_ctx_create(device, nullptr, &c) != TW_OK)
            throw std::runtime_error("twoway: no CUDA device available for the B200 path");
        slot.reset(c);
    }
    return slot.get();
}

// 64-bit mix over the topology and masses: a changed MeshState re-uploads.
// Eight independent multiply lanes over 64-byte blocks (the chains overlap):
// the bow knot's 4 MB of topology hash in ~0.3 ms per call instead of ~1.3 ms.
inline uint64_t topology_hash(const MeshState& m) {
    uint64_t h = 0x9e3779b97f4a7c15ull ^ static_cast<uint64_t>(m.positions.size());
    auto mix = [&h](const void* p, size_t bytes) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        uint64_t l[8];
        for (int k = 0; k < 8; ++k) l[k] = h ^ (0x243f6a8885a308d3ull * static_cast<uint64_t>(k + 1));
        size_t i = 0;
        for (; i + 64 <= bytes; i += 64) {
            uint64_t w[8];
            std::memcpy(w, b + i, 64);
#pragma GCC unroll 8
            for (int k = 0; k < 8; ++k) l[k] = (l[k] ^ w[k]) * 0xff51afd7ed558ccdull;
        }
        for (int k = 0; k < 8; ++k) h = (h ^ l[k] ^ (l[k] >> 29)) * 0xc4ceb9fe1a85ec53ull, h ^= h >> 31;
        for (; i < bytes; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
        h ^= bytes;
    };
    mix(m.edges.data(), m.edges.size() * sizeof(m.edges[0]));
    mix(m.triangles.data(), m.triangles.size() * sizeof(m.triangles[0]));
    mix(m.inv_mass.data(), m.inv_mass.size() * sizeof(double));
    return h;
}

// The finalized edge list goes in as explicit edges (finalize is idempotent
// on it), so the device edge indices are the MeshState's.
inline tw_mesh* device_mesh(tw_ctx* ctx, int device, const MeshState& mesh) {
    const uint64_t h = topology_hash(mesh);
    Runtime::Upload& up = runtime().uploads[{device, &mesh}];
    if (up.mesh && up.hash == h) return up.mesh.get();
    std::vector<int32_t> e, t;
    e.reserve(2 * mesh.edges.size());
    t.reserve(3 * mesh.triangles.size());
    for (const auto& ed : mesh.edges) e.insert(e.end(), {ed[0], ed[1]});
    for (const auto& tr : mesh.triangles) t.insert(t.end(), {tr[0], tr[1], tr[2]});
    tw_mesh* m = nullptr;
    check(tw_mesh_create(ctx, mesh.num_vertices(), mesh.inv_mass.empty() ? nullptr : mesh.inv_mass.data(),
                         static_cast<int32_t>(mesh.edges.size()), e.data(), 0, nullptr,
                         static_cast<int32_t>(mesh.triangles.size()), t.data(), &m),
          ctx);
    up.mesh.reset(m);
    up.hash = h;
    return m;
}

// A vertex-only device mesh (rows that carry their own vertex ids).
inline MeshPtr vertex_mesh(tw_ctx* ctx, std::span<const double> inv_mass) {
    tw_mesh* m = nullptr;
    check(tw_mesh_create(ctx, static_cast<int32_t>(inv_mass.size()), inv_mass.data(), 0, nullptr, 0, nullptr, 0,
                         nullptr, &m),
          ctx);
    return MeshPtr(m);
}

inline std::vector<double> flatten(PositionsView p) {
    std::vector<double> f(3 * p.size());
    for (size_t i = 0; i < p.size(); ++i)
        for (int k = 0; k < 3; ++k) f[3 * i + k] = p[i][k];
    return f;
}

inline Positions unflatten(const double* f, size_t n) {
    Positions p(n);
    for (size_t i = 0; i < n; ++i) p[i] = Vec3(f[3 * i], f[3 * i + 1], f[3 * i + 2]);
    return p;
}

}  // namespace twoway::detail
