// fl_api.cu -- C-ABI entry points of libfemlite_b200 (include/femlite_b200.h).
//
// Host-side orchestration only: argument checks mirroring the reference's
// errors, device buffer management, staging of host arrays, launches on the
// context stream, and the deferred error report in fl_result_sizes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fl_internal.cuh"
#include "fl_kernels.cuh"

namespace fl {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int DevBuf::ensure(size_t n) {
    if (n == 0) n = 16;
    if (n <= bytes) return FL_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) {
        p = nullptr;
        cudaGetLastError();
        return set_error(FL_ERR_OUT_OF_MEMORY,
                         "cudaMalloc(" + std::to_string(n) + "): " + cudaGetErrorString(e));
    }
    bytes = n;
    return FL_OK;
}

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

static bool field_ok(const fl_field* f) {
    if (!f) return true;
    switch (f->kind) {
    case FL_FIELD_NONE:
    case FL_FIELD_CONST:
    case FL_FIELD_SINSIN:
    case FL_FIELD_X:
    case FL_FIELD_XYZ:
    case FL_FIELD_COEF_C5: return true;
    case FL_FIELD_SAMPLES: return f->samples != nullptr || f->n_samples == 0;
    }
    return false;
}

// Device view of a field; host samples are staged into `stage`.
static int field_desc(fl_ctx* ctx, const fl_field* f, int64_t expected, DevBuf& stage,
                      FieldDesc* out, const char* what) {
    out->kind = f ? f->kind : FL_FIELD_NONE;
    out->value = f ? f->value : 0.0;
    out->samples = nullptr;
    if (!f || f->kind != FL_FIELD_SAMPLES) return FL_OK;
    if (f->n_samples != expected)
        return set_error(FL_E_SHAPE_MISMATCH, std::string(what) + ": expected " +
                                                  std::to_string(expected) + " samples, got " +
                                                  std::to_string(f->n_samples));
    if (f->mem == FL_MEM_DEVICE) {
        out->samples = f->samples;
        return FL_OK;
    }
    FL_TRY(stage.ensure(sizeof(double) * (size_t)std::max<int64_t>(expected, 1)));
    if (expected > 0)
        FL_CUDA(cudaMemcpyAsync(stage.p, f->samples, sizeof(double) * (size_t)expected,
                                cudaMemcpyHostToDevice, ctx->stream));
    out->samples = stage.as<double>();
    return FL_OK;
}

static int copy_in(fl_ctx* ctx, DevBuf& dst, const void* src, size_t bytes, int mem) {
    FL_TRY(dst.ensure(bytes));
    if (bytes == 0) return FL_OK;
    if (!src) return set_error(FL_ERR_ARGUMENT, "null input array");
    FL_CUDA(cudaMemcpyAsync(dst.p, src, bytes,
                            mem == FL_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            ctx->stream));
    return FL_OK;
}

struct ResultStage {
    DevBuf f, coef, g_dir, g_neu, sub[6];
};

}  // namespace fl

using namespace fl;

// result-owned staging lives next to the result (kept out of the public struct)
struct fl_result_ext {
    ResultStage stage;
    bool g_missing = false;
    bool partition_done = false;
    // last column launch, kept for the general-kernel fallback
    ColParams last{};
    fl_mesh* last_mesh = nullptr;
    bool last_valid = false;
};

// Re-run the column pass on the general warp-per-column kernel (a tile or a
// column exceeded the tiled kernel's shared-memory limits).
static int rerun_general(fl_result* res, fl_result_ext* x) {
    fl_ctx* ctx = res->ctx;
    fl_mesh* mesh = x->last_mesh;
    ColParams p = x->last;
    uint32_t* counters = res->counters.as<uint32_t>();
    if (res->v4_used) {
        // the label-space pass overflowed: the general kernel works on the
        // id-space plan and writes every output in node order itself
        if (!mesh->planned || mesh->stats_stale) FL_TRY(fl_mesh_plan(ctx, mesh));
        p.inc_ptr = mesh->inc_ptr.as<int32_t>();
        p.inc = mesh->inc.as<uint32_t>();
        p.lcnt = nullptr;
        p.nadd = nullptr;  // the general kernel forms the Neumann shares itself
        res->v4_used = false;
    }
    // the general kernel may need the plan's full output bound
    const size_t cap = (size_t)std::max<int64_t>(mesh->nnz_bound, 1);
    if (p.want_a) {
        FL_TRY(res->arr[FL_A_ROW_IDX].ensure(sizeof(int32_t) * cap));
        FL_TRY(res->arr[FL_A_VALUES].ensure(sizeof(double) * cap));
        p.row_idx = res->arr[FL_A_ROW_IDX].as<int32_t>();
        p.values = res->arr[FL_A_VALUES].as<double>();
        p.cap_a = (int64_t)cap;
    }
    if (p.want_sys) {
        FL_TRY(res->arr[FL_AFF_ROW_IDX].ensure(sizeof(int32_t) * cap));
        FL_TRY(res->arr[FL_AFF_VALUES].ensure(sizeof(double) * cap));
        p.ff_row_idx = res->arr[FL_AFF_ROW_IDX].as<int32_t>();
        p.ff_values = res->arr[FL_AFF_VALUES].as<double>();
        p.cap_ff = (int64_t)cap;
    }
    FL_TRY(launch_inc_sort(ctx, mesh));
    FL_CUDA(cudaMemsetAsync(counters + CNT_TICKET, 0, sizeof(uint32_t), ctx->stream));
    FL_CUDA(cudaMemsetAsync(counters + CNT_ERR, 0, sizeof(uint32_t), ctx->stream));
    const int tw = column_tile_width();
    p.n_tiles = (p.n_cols + tw - 1) / tw;
    FL_CUDA(cudaMemsetAsync(res->tile_status.p, 0, sizeof(uint64_t) * ((size_t)p.n_tiles + 1),
                            ctx->stream));
    FL_TRY(launch_columns(ctx, mesh->dim, p));
    return FL_OK;
}
static fl_result_ext* ext_of(fl_result* r) {
    return reinterpret_cast<fl_result_ext*>(reinterpret_cast<char*>(r) + sizeof(fl_result));
}

extern "C" {

FL_API int fl_abi_version(void) { return FL_ABI_VERSION; }

FL_API const char* fl_last_error(void) { return g_last_error.c_str(); }

FL_API int fl_create(int device, fl_ctx** out) {
    if (!out) return set_error(FL_ERR_ARGUMENT, "out is null");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return set_error(FL_ERR_NO_DEVICE, std::string("no CUDA device: ") +
                                               (e != cudaSuccess ? cudaGetErrorString(e) : "count 0"));
    }
    if (device < 0 || device >= count) return set_error(FL_ERR_ARGUMENT, "bad device ordinal");
    FL_CUDA(cudaSetDevice(device));
    fl_ctx* ctx = new fl_ctx();
    ctx->device = device;
    cudaDeviceProp prop{};
    FL_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
        delete ctx;
        return set_error(FL_ERR_UNSUPPORTED, std::string("libfemlite_b200 is built for sm_100a; device is ") +
                                                 prop.name);
    }
    ctx->sm_count = prop.multiProcessorCount;
    FL_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    FL_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    FL_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    FL_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    const char* ov = std::getenv("FL_OVERLAP");
    ctx->overlap = !(ov && ov[0] == '0');
    FL_CUDA(cudaMallocHost(&ctx->pinned, 4096));
    FL_TRY(v4_init_consts(ctx));
    const char* prof = std::getenv("FL_PROFILE");
    ctx->profile = prof && prof[0] == '1';
    if (ctx->profile)
        for (auto& ev : ctx->ev) FL_CUDA(cudaEventCreate(&ev));
    const char* ph = std::getenv("FL_PHASES");
    ctx->phase_timing = ph && ph[0] == '1';
    if (ctx->phase_timing) FL_TRY(ctx->phases.ensure(sizeof(unsigned long long) * 8));
    *out = ctx;
    return FL_OK;
}

FL_API int fl_destroy(fl_ctx* ctx) {
    if (!ctx) return FL_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->aux_stream) {
        cudaStreamSynchronize(ctx->aux_stream);
        cudaStreamDestroy(ctx->aux_stream);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    ctx->scan_ws.release();
    ctx->scan_ws_aux.release();
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->profile)
        for (auto& ev : ctx->ev) cudaEventDestroy(ev);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return FL_OK;
}

FL_API int fl_set_stream(fl_ctx* ctx, void* stream) {
    if (!ctx) return set_error(FL_ERR_ARGUMENT, "ctx is null");
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return FL_OK;
}

FL_API int fl_synchronize(fl_ctx* ctx) {
    if (!ctx) return set_error(FL_ERR_ARGUMENT, "ctx is null");
    FL_CUDA(cudaStreamSynchronize(ctx->stream));
    return FL_OK;
}

FL_API int64_t fl_launch_count(const fl_ctx* ctx) { return ctx ? ctx->launches : -1; }

FL_API int fl_last_timings(const fl_ctx* ctx, double* ms4) {
    if (!ctx || !ms4) return set_error(FL_ERR_ARGUMENT, "null argument");
    for (int i = 0; i < 4; ++i) ms4[i] = ctx->timings[i];
    return FL_OK;
}

FL_API int fl_last_kernel_timings(const fl_ctx* ctx, double* ms3) {
    if (!ctx || !ms3) return set_error(FL_ERR_ARGUMENT, "null argument");
    for (int i = 0; i < 3; ++i) ms3[i] = ctx->ktimings[i];
    return FL_OK;
}

// ---- mesh -----------------------------------------------------------------------
FL_API int fl_mesh_create(fl_ctx* ctx, int dim, int32_t n_nodes, int32_t n_elems,
                          const double* nodes, const int32_t* elems, const int8_t* bd_flags,
                          int mem, fl_mesh** out) {
    if (!ctx || !out) return set_error(FL_ERR_ARGUMENT, "null argument");
    *out = nullptr;
    if (dim != 2 && dim != 3)
        return set_error(FL_E_INVALID_PARAMETER, "mesh dimension must be 2 or 3");
    if (n_nodes < 0 || n_elems < 0) return set_error(FL_E_SHAPE_MISMATCH, "negative size");
    // incidence keys pack (j << 30 | t): element ids must fit 30 bits
    if (n_elems >= (1 << 30) || (int64_t)n_elems * (dim + 1) > INT32_MAX)
        return set_error(FL_ERR_UNSUPPORTED, "more than 2^30 elements is not supported");
    FL_CUDA(cudaSetDevice(ctx->device));
    fl_mesh* m = new fl_mesh();
    m->ctx = ctx;
    m->dim = dim;
    m->n_nodes = n_nodes;
    m->n_elems = n_elems;
    m->col_begin = 0;
    m->col_end = n_nodes;
    const size_t nv = (size_t)dim + 1;
    int rc = copy_in(ctx, m->nodes, nodes, sizeof(double) * (size_t)n_nodes * dim, mem);
    if (!rc) rc = copy_in(ctx, m->elems, elems, sizeof(int32_t) * (size_t)n_elems * nv, mem);
    if (!rc && bd_flags) {
        rc = copy_in(ctx, m->flags, bd_flags, (size_t)n_elems * nv, mem);
        m->has_flags = true;
    }
    if (!rc && !bd_flags) rc = m->flags.ensure(16);
    if (rc) {
        fl_mesh_destroy(m);
        return rc;
    }
    *out = m;
    return FL_OK;
}

FL_API int fl_mesh_set_nodes(fl_ctx* ctx, fl_mesh* mesh, const double* nodes, int mem) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    mesh->n_bfaces = -1;
    return copy_in(ctx, mesh->nodes, nodes, sizeof(double) * (size_t)mesh->n_nodes * mesh->dim, mem);
}

FL_API int fl_mesh_set_flags(fl_ctx* ctx, fl_mesh* mesh, const int8_t* bd_flags, int mem) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (!bd_flags) {
        mesh->has_flags = false;
        return FL_OK;
    }
    mesh->has_flags = true;
    return copy_in(ctx, mesh->flags, bd_flags, (size_t)mesh->n_elems * (mesh->dim + 1), mem);
}

FL_API int fl_mesh_set_elems(fl_ctx* ctx, fl_mesh* mesh, const int32_t* elems, int mem) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    mesh->n_bfaces = -1;
    mesh->planned = false;
    mesh->lp.planned = false;
    return copy_in(ctx, mesh->elems, elems, sizeof(int32_t) * (size_t)mesh->n_elems * (mesh->dim + 1),
                   mem);
}

FL_API int fl_mesh_set_columns(fl_ctx* ctx, fl_mesh* mesh, int32_t col_begin, int32_t col_end) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (col_begin < 0 || col_end < col_begin || col_end > mesh->n_nodes)
        return set_error(FL_E_INDEX_OUT_OF_RANGE, "column range outside [0, n_nodes]");
    if (col_begin != mesh->col_begin || col_end != mesh->col_end) {
        mesh->planned = false;
        mesh->lp.planned = false;  // the label plan orders the owned columns first
        mesh->lp.ever = false;     // and its bounds are the old range's: plan synchronously
    }
    mesh->col_begin = col_begin;
    mesh->col_end = col_end;
    return FL_OK;
}

// ---- boundary faces (set_boundary_flags, mesh.hpp:251-304) ---------------------------
FL_API int fl_boundary_faces(fl_ctx* ctx, fl_mesh* mesh, int64_t* n_faces) {
    if (!ctx || !mesh || !n_faces) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (mesh->col_begin != 0 || mesh->col_end != mesh->n_nodes)
        return set_error(FL_ERR_ARGUMENT, "boundary faces need the whole mesh (no column range)");
    FL_CUDA(cudaSetDevice(ctx->device));
    if (!mesh->planned || mesh->stats_stale) FL_TRY(fl_mesh_plan(ctx, mesh));
    return launch_boundary_faces(ctx, mesh, n_faces);
}

FL_API int fl_boundary_faces_copy(fl_ctx* ctx, fl_mesh* mesh, int32_t* faces, double* centroids,
                                  int mem) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (mesh->n_bfaces < 0) return set_error(FL_ERR_ARGUMENT, "call fl_boundary_faces first");
    const size_t nb = (size_t)mesh->n_bfaces;
    const cudaMemcpyKind kind = mem == FL_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (faces && nb) FL_CUDA(cudaMemcpyAsync(faces, mesh->bfaces.p, sizeof(int32_t) * 2 * nb, kind, ctx->stream));
    if (centroids && nb)
        FL_CUDA(cudaMemcpyAsync(centroids, mesh->bcent.p, sizeof(double) * 3 * nb, kind, ctx->stream));
    if (mem != FL_MEM_DEVICE) FL_CUDA(cudaStreamSynchronize(ctx->stream));
    return FL_OK;
}

FL_API int fl_mesh_set_boundary_flags(fl_ctx* ctx, fl_mesh* mesh, const int8_t* face_flags,
                                      int8_t fill, int mem) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (mesh->n_bfaces < 0) return set_error(FL_ERR_ARGUMENT, "call fl_boundary_faces first");
    const int8_t* vals = nullptr;
    if (face_flags) {
        FL_TRY(copy_in(ctx, mesh->bstage, face_flags, (size_t)mesh->n_bfaces, mem));
        vals = mesh->bstage.as<int8_t>();
    }
    return launch_boundary_scatter(ctx, mesh, vals, fill);
}

FL_API int fl_mesh_destroy(fl_mesh* mesh) {
    if (!mesh) return FL_OK;
    if (mesh->ctx) cudaStreamSynchronize(mesh->ctx->stream);
    mesh->nodes.release();
    mesh->elems.release();
    mesh->flags.release();
    mesh->inc_ptr.release();
    mesh->inc.release();
    mesh->cursor.release();
    mesh->emark.release();
    mesh->bmark.release();
    mesh->bpos.release();
    mesh->bfaces.release();
    mesh->bcent.release();
    mesh->bstage.release();
    mesh->bcnt.release();
    mesh->stats.release();
    auto& lp = mesh->lp;
    for (fl::DevBuf* b : {&lp.lab, &lp.lptr, &lp.linc, &lp.lel, &lp.misc, &lp.cells, &lp.stage})
        b->release();
    delete mesh;
    return FL_OK;
}

static int read_err_word(fl_ctx* ctx, uint32_t* d_word, uint32_t* host) {
    FL_CUDA(cudaMemcpyAsync(ctx->pinned, d_word, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    FL_CUDA(cudaStreamSynchronize(ctx->stream));
    *host = *static_cast<uint32_t*>(ctx->pinned);
    return FL_OK;
}

FL_API int fl_mesh_validate(fl_ctx* ctx, fl_mesh* mesh) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_TRY(mesh->stats.ensure(sizeof(unsigned long long) * 4));
    uint32_t* d_err = reinterpret_cast<uint32_t*>(mesh->stats.as<unsigned long long>() + 3);
    FL_CUDA(cudaMemsetAsync(d_err, 0, sizeof(uint32_t), ctx->stream));
    FL_TRY(launch_validate(ctx, mesh, d_err));
    uint32_t e = 0;
    FL_TRY(read_err_word(ctx, d_err, &e));
    // make_mesh order: index range and flag values (check_arrays), then measures
    if (e & DERR_INDEX) return set_error(FL_E_INDEX_OUT_OF_RANGE, "element vertex index out of range");
    if (e & DERR_FLAG) return set_error(FL_E_INVALID_FLAG_VALUE, "boundary flag not in {0,1,2,3}");
    if (e & DERR_MEASURE)
        return set_error(FL_E_NON_POSITIVE_VOLUME, "element has non-positive signed measure");
    return FL_OK;
}

FL_API int fl_mesh_plan(fl_ctx* ctx, fl_mesh* mesh) {
    if (!ctx || !mesh) return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_CUDA(cudaSetDevice(ctx->device));
    FL_TRY(mesh->stats.ensure(sizeof(unsigned long long) * 4));
    uint32_t* d_err = reinterpret_cast<uint32_t*>(mesh->stats.as<unsigned long long>() + 3);
    FL_TRY(launch_plan_kernels(ctx, mesh, d_err));  // zeroes stats (incl. the error word)
    FL_CUDA(cudaMemcpyAsync(ctx->pinned, mesh->stats.p, sizeof(unsigned long long) * 4,
                            cudaMemcpyDeviceToHost, ctx->stream));
    FL_CUDA(cudaStreamSynchronize(ctx->stream));
    const unsigned long long* st = static_cast<const unsigned long long*>(ctx->pinned);
    const uint32_t e = static_cast<uint32_t>(st[3] & 0xFFFFFFFFull);
    if (e & DERR_INDEX) return set_error(FL_E_INDEX_OUT_OF_RANGE, "element vertex index out of range");
    mesh->nnz_bound = (int64_t)st[0];
    mesh->max_inc = (int32_t)st[1];
    mesh->planned = true;
    mesh->ever_planned = true;
    mesh->stats_stale = false;
    return FL_OK;
}

// ---- results ----------------------------------------------------------------------
FL_API int fl_result_create(fl_ctx* ctx, fl_result** out) {
    if (!ctx || !out) return set_error(FL_ERR_ARGUMENT, "null argument");
    void* raw = ::operator new(sizeof(fl_result) + sizeof(fl_result_ext));
    fl_result* r = new (raw) fl_result();
    new (ext_of(r)) fl_result_ext();
    r->ctx = ctx;
    int rc = r->counters.ensure(sizeof(uint32_t) * CNT_WORDS);
    if (rc) {
        fl_result_destroy(r);
        return rc;
    }
    *out = r;
    return FL_OK;
}

FL_API int fl_result_destroy(fl_result* r) {
    if (!r) return FL_OK;
    if (r->ctx) cudaStreamSynchronize(r->ctx->stream);
    for (auto& a : r->arr) a.release();
    r->is_dir.release();
    r->is_neu.release();
    r->fidx.release();
    r->tile_status.release();
    for (auto& b : r->stage) b.release();
    r->tile_tot.release();
    r->tile_off.release();
    r->colcnt.release();
    for (auto& b : r->erec) b.release();
    for (auto& b : r->hyb) b.release();
    for (auto& b : r->v4) b.release();
    r->counters.release();
    fl_result_ext* x = ext_of(r);
    x->stage.f.release();
    x->stage.coef.release();
    x->stage.g_dir.release();
    x->stage.g_neu.release();
    for (auto& s : x->stage.sub) s.release();
    x->~fl_result_ext();
    r->~fl_result();
    ::operator delete(static_cast<void*>(r));
    return FL_OK;
}

FL_API int fl_assemble(fl_ctx* ctx, fl_mesh* mesh, const fl_field* f, const fl_field* coef,
                       const fl_field* g_dirichlet, const fl_field* g_neumann, uint32_t what,
                       fl_result* res) {
    if (!ctx || !mesh || !res) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (!field_ok(f) || !field_ok(coef) || !field_ok(g_dirichlet) || !field_ok(g_neumann))
        return set_error(FL_ERR_ARGUMENT, "invalid field descriptor");
    const bool replan = what & FL_REPLAN;
    what &= ~(uint32_t)FL_REPLAN;
    if (what & FL_OUT_SYSTEM) what |= FL_OUT_STIFFNESS | FL_OUT_LOAD | FL_OUT_PARTITION;
    if (what == 0) return set_error(FL_ERR_ARGUMENT, "nothing requested");
    FL_CUDA(cudaSetDevice(ctx->device));
    const cudaStream_t s = ctx->stream;
    if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[0], s));
    ctx->plan_timed = false;
    ctx->kernel_timed = false;
    const bool need_plan = what & (FL_OUT_STIFFNESS | FL_OUT_LOAD);
    const char* kern = std::getenv("FL_KERNEL");
    const char kk = kern ? kern[0] : '0';
    // the label-space pipeline (fl_columns4.cu) takes every mesh (whole or a
    // column range) whose valence fits its kernel; FL_V4=0 forces the id-space one
    const char* v4env = std::getenv("FL_V4");
    bool use_v4 = need_plan && kk == '0' && !(v4env && v4env[0] == '0') && mesh->n_nodes > 0 &&
                  mesh->n_elems > 0 && mesh->lp.ok;
    // An asynchronous label re-plan (previous bounds known) is independent of the
    // partition + FaceLists pass: it is launched after them, which run on the
    // side stream beside it (below).
    const bool defer_plan = use_v4 && (replan || !mesh->lp.planned) && mesh->lp.ever && ctx->overlap &&
                            (what & FL_OUT_PARTITION);
    if (use_v4 && (replan || !mesh->lp.planned) && !defer_plan) {
        // a re-plan runs asynchronously with the previous bounds (fl_result_sizes
        // refreshes them and reruns on the general kernel if they were exceeded)
        FL_TRY(v4_plan(ctx, mesh, !mesh->lp.ever));
        ctx->plan_timed = true;
        if (!mesh->lp.ok) use_v4 = false;  // valence above the kernel's lanes
    }
    if (use_v4) {
    } else if (need_plan && (replan || !mesh->planned) && mesh->ever_planned) {
        // Rebuild asynchronously: allocation and kernel choice use the previous
        // plan's bounds; fl_result_sizes refreshes the statistics and, should the
        // new topology exceed them, re-runs the column pass on the general kernel.
        uint32_t* d_err = reinterpret_cast<uint32_t*>(mesh->stats.as<unsigned long long>() + 3);
        FL_TRY(launch_plan_kernels(ctx, mesh, d_err));
        mesh->planned = true;
        mesh->stats_stale = true;
        ctx->plan_timed = true;
    } else if (need_plan && !mesh->planned) {
        FL_TRY(fl_mesh_plan(ctx, mesh));
        ctx->plan_timed = true;
    }
    if (ctx->profile && !defer_plan) FL_CUDA(cudaEventRecord(ctx->ev[1], s));
    fl_result_ext* x = ext_of(res);
    res->sizes_valid = false;
    res->v4_used = false;
    res->what = what;
    const int32_t N = mesh->n_nodes;
    const int32_t C0 = mesh->col_begin, NC = mesh->col_end - mesh->col_begin;
    res->n = NC;
    res->m = N;
    res->col_begin = C0;
    res->dim = mesh->dim;
    const int64_t NT = mesh->n_elems;
    const int nv = mesh->dim + 1;
    const bool want_a = what & FL_OUT_STIFFNESS, want_b = what & FL_OUT_LOAD;
    const bool want_p = what & FL_OUT_PARTITION, want_sys = what & FL_OUT_SYSTEM;

    ColParams p{};
    FL_TRY(field_desc(ctx, f, NT * nv, x->stage.f, &p.f, "f"));
    FL_TRY(field_desc(ctx, coef, NT, x->stage.coef, &p.coef, "coefficient"));
    FL_TRY(field_desc(ctx, g_dirichlet, N, x->stage.g_dir, &p.g_dir, "g_dirichlet"));
    FL_TRY(field_desc(ctx, g_neumann, NT * nv, x->stage.g_neu, &p.g_neu, "g_neumann"));
    x->g_missing = want_sys && p.g_dir.kind == FL_FIELD_NONE;

    // outputs (column-indexed ones hold the owned range only)
    const size_t n1 = (size_t)N + 1, nc1 = (size_t)NC + 1;
    // Output capacity.  The tiled / register kernels keep at most 12 (2-D) /
    // 24 (3-D) distinct rows per column (else they flag the general kernel,
    // which re-sizes to the plan's bound in rerun_general): size for that.
    const int64_t fast_rows = mesh->dim == 2 ? 12 : 24;
    const int64_t bound = std::max<int64_t>(use_v4 ? mesh->lp.nnz_bound : mesh->nnz_bound, 1);
    // columns above the register kernel's valence go to the hybrid pass, sized
    // by the plan's bound
    const bool hyb = !use_v4 && mesh->max_inc > columns3_lanes(mesh->dim, mesh->max_inc);
    const size_t cap = (size_t)(kk == '1' || hyb ? bound
                                                 : std::min<int64_t>(bound, fast_rows * std::max(NC, 1)));
    uint32_t* counters = res->counters.as<uint32_t>();
    FL_CUDA(cudaMemsetAsync(counters, 0, sizeof(uint32_t) * CNT_WORDS, s));
    if (want_a) {
        FL_TRY(res->arr[FL_A_COL_PTR].ensure(sizeof(int32_t) * nc1));
        FL_TRY(res->arr[FL_A_ROW_IDX].ensure(sizeof(int32_t) * cap));
        FL_TRY(res->arr[FL_A_VALUES].ensure(sizeof(double) * cap));
        FL_CUDA(cudaMemsetAsync(res->arr[FL_A_COL_PTR].p, 0, sizeof(int32_t) * nc1, s));
    }
    if (want_b) FL_TRY(res->arr[FL_B].ensure(sizeof(double) * nc1));
    if (want_p) {
        FL_TRY(res->is_dir.ensure(n1));
        FL_TRY(res->is_neu.ensure(n1));
        FL_TRY(res->fidx.ensure(sizeof(int32_t) * 2 * n1));
        FL_TRY(res->arr[FL_DIR_NODES].ensure(sizeof(int32_t) * n1));
        FL_TRY(res->arr[FL_FREE_NODES].ensure(sizeof(int32_t) * n1));
    }
    if (want_sys) {
        FL_TRY(res->arr[FL_U0].ensure(sizeof(double) * nc1));
        FL_TRY(res->arr[FL_B_MOD].ensure(sizeof(double) * nc1));
        FL_TRY(res->arr[FL_B_F].ensure(sizeof(double) * nc1));
        FL_TRY(res->arr[FL_AFF_COL_PTR].ensure(sizeof(int32_t) * nc1));
        FL_TRY(res->arr[FL_AFF_ROW_IDX].ensure(sizeof(int32_t) * cap));
        FL_TRY(res->arr[FL_AFF_VALUES].ensure(sizeof(double) * cap));
        FL_CUDA(cudaMemsetAsync(res->arr[FL_AFF_COL_PTR].p, 0, sizeof(int32_t), s));
    }
    if (defer_plan) {
        // fork: partition + FaceLists on the side stream (their own scan workspace),
        // the label plan on the main one; join before the column pass
        FL_CUDA(cudaEventRecord(ctx->ev_fork, s));
        FL_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->ev_fork, 0));
        ctx->stream = ctx->aux_stream;
        std::swap(ctx->scan_ws, ctx->scan_ws_aux);
        int rc = launch_partition(ctx, mesh, res);
        if (rc == FL_OK) rc = launch_face_lists(ctx, mesh, res);
        std::swap(ctx->scan_ws, ctx->scan_ws_aux);
        ctx->stream = s;
        cudaEventRecord(ctx->ev_join, ctx->aux_stream);
        if (rc == FL_OK) rc = v4_plan(ctx, mesh, false);
        cudaStreamWaitEvent(s, ctx->ev_join, 0);  // join (also on failure: the side stream never runs ahead)
        if (rc != FL_OK) return rc;
        ctx->plan_timed = true;
        if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[1], s));
    } else if (want_p) {
        FL_TRY(launch_partition(ctx, mesh, res));
        FL_TRY(launch_face_lists(ctx, mesh, res));
    }
    if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[2], s));

    if (want_a || want_b) {
        const int tw = column_tile_width();
        p.n_nodes = N;
        p.n_elems = (int32_t)NT;
        p.c_begin = C0;
        p.n_cols = NC;
        p.n_tiles = (NC + tw - 1) / tw;
        FL_TRY(res->tile_status.ensure(sizeof(uint64_t) * ((size_t)p.n_tiles + 1)));
        FL_CUDA(cudaMemsetAsync(res->tile_status.p, 0, sizeof(uint64_t) * ((size_t)p.n_tiles + 1), s));
        p.nodes = mesh->nodes.as<double>();
        p.elems = mesh->elems.as<int32_t>();
        p.flags = mesh->flags.as<int8_t>();
        p.inc_ptr = mesh->inc_ptr.as<int32_t>();
        p.inc = mesh->inc.as<uint32_t>();
        p.want_a = want_a;
        p.want_b = want_b;
        p.want_sys = want_sys;
        p.need_lift = want_sys && !(p.g_dir.kind == FL_FIELD_NONE ||
                                    (p.g_dir.kind == FL_FIELD_CONST && p.g_dir.value == 0.0));
        p.has_neumann = want_b && mesh->has_flags && want_p;
        if (want_b && !want_p && mesh->has_flags && g_neumann && g_neumann->kind != FL_FIELD_NONE) {
            // Neumann data needs the flag-2 node marks: run the marking pass too.
            FL_TRY(res->is_dir.ensure(n1));
            FL_TRY(res->is_neu.ensure(n1));
            FL_TRY(res->fidx.ensure(sizeof(int32_t) * 2 * n1));
            FL_TRY(res->arr[FL_DIR_NODES].ensure(sizeof(int32_t) * n1));
            FL_TRY(res->arr[FL_FREE_NODES].ensure(sizeof(int32_t) * n1));
            FL_TRY(launch_partition(ctx, mesh, res));
            p.has_neumann = true;
        }
        p.is_dir = res->is_dir.as<int8_t>();
        p.is_neu = res->is_neu.as<int8_t>();
        p.fidx = res->fidx.as<int32_t>();
        p.emark = NC < N ? mesh->emark.as<uint8_t>() : nullptr;
        // free nodes below the range = free_rank[C0] (k_partition's exclusive scan)
        p.f_begin = (C0 > 0 && want_sys) ? res->fidx.as<int32_t>() + n1 + C0 : nullptr;
        p.col_ptr = res->arr[FL_A_COL_PTR].as<int32_t>();
        p.row_idx = res->arr[FL_A_ROW_IDX].as<int32_t>();
        p.values = res->arr[FL_A_VALUES].as<double>();
        p.b = res->arr[FL_B].as<double>();
        p.u0 = res->arr[FL_U0].as<double>();
        p.b_mod = res->arr[FL_B_MOD].as<double>();
        p.ff_col_ptr = res->arr[FL_AFF_COL_PTR].as<int32_t>();
        p.ff_row_idx = res->arr[FL_AFF_ROW_IDX].as<int32_t>();
        p.ff_values = res->arr[FL_AFF_VALUES].as<double>();
        p.b_f = res->arr[FL_B_F].as<double>();
        p.tile_status = res->tile_status.as<uint64_t>();
        p.ticket = counters + CNT_TICKET;
        p.err = counters + CNT_ERR;
        p.cap_a = want_a ? (int64_t)cap : 0;
        p.cap_ff = want_sys ? (int64_t)cap : 0;
        p.phase_cycles = nullptr;
        if (ctx->phase_timing) {
            p.phase_cycles = ctx->phases.as<unsigned long long>();
            FL_CUDA(cudaMemsetAsync(p.phase_cycles, 0, sizeof(unsigned long long) * 8, s));
        }
        // a cached plan used again: sort its segments once, the register kernel
        // then skips its key sort on this and every later assembly of the mesh
        const char* ks = std::getenv("FL_KEYSORT");
        if (kk == '0' && !use_v4 && !ctx->plan_timed && !(ks && ks[0] == '0')) {
            if (!mesh->inc_sorted) FL_TRY(launch_inc_sort(ctx, mesh));
            p.keys_sorted = true;
        }
        x->last = p;
        x->last_mesh = mesh;
        x->last_valid = true;
        if (NC > 0) {
            // element records + v3 (register-centric) by default; v2 (tiled)
            // carries the Dirichlet lift; v1 (general) is the fallback.
            // FL_KERNEL=1|2|3 forces one (3 = v3 with in-kernel geometry).
            const char k = kk;
            if (use_v4) {
                FL_TRY(v4_columns(ctx, mesh, p, res));
                x->last = p;
            } else if (k == '1') {
                FL_TRY(launch_inc_sort(ctx, mesh));
                FL_TRY(launch_columns(ctx, mesh->dim, p));
            } else if (k == '2' || (k == '3' && (p.need_lift || (p.has_neumann && p.g_neu.kind != FL_FIELD_NONE)))) {
                FL_TRY(launch_columns2(ctx, mesh->dim, p, mesh->max_inc, res));
            } else {
                // Neumann data: per-node shares first, added by the register kernel
                if (p.want_b && p.has_neumann && p.g_neu.kind != FL_FIELD_NONE)
                    FL_TRY(launch_neumann_add(ctx, mesh->dim, p, res));
                if (mesh->max_inc > columns3_lanes(mesh->dim, mesh->max_inc))
                    FL_TRY(launch_hybrid(ctx, mesh->dim, p, mesh, res, k != '3'));
                else
                    FL_TRY(launch_columns3(ctx, mesh->dim, p, mesh->max_inc, res, k != '3'));
            }
        }
    }
    if (ctx->profile) {
        FL_CUDA(cudaEventRecord(ctx->ev[3], s));
        ctx->timing_pending = true;
    }
    return FL_OK;
}

FL_API int fl_result_sizes(fl_result* res, fl_sizes* out) {
    if (!res || !out) return set_error(FL_ERR_ARGUMENT, "null argument");
    fl_ctx* ctx = res->ctx;
    fl_result_ext* x = ext_of(res);
    if (!res->sizes_valid) {
        const cudaStream_t s = ctx->stream;
        uint32_t* h = static_cast<uint32_t*>(ctx->pinned);
        FL_CUDA(cudaMemcpyAsync(h, res->counters.p, sizeof(uint32_t) * CNT_WORDS,
                                cudaMemcpyDeviceToHost, s));
        int32_t* hn = reinterpret_cast<int32_t*>(h + CNT_WORDS);
        hn[0] = hn[1] = hn[2] = hn[3] = hn[4] = 0;
        fl_mesh* lm = x->last_valid ? x->last_mesh : nullptr;
        unsigned long long* hst = reinterpret_cast<unsigned long long*>(h + CNT_WORDS + 16);
        if (lm && lm->stats_stale && !res->v4_used)
            FL_CUDA(cudaMemcpyAsync(hst, lm->stats.p, sizeof(unsigned long long) * 4,
                                    cudaMemcpyDeviceToHost, s));
        // the label plan's statistics and error word (v4 re-plans run asynchronously)
        const bool v4s = lm && res->v4_used && lm->lp.stale;
        unsigned long long* h4 = reinterpret_cast<unsigned long long*>(static_cast<char*>(ctx->pinned) + 256);
        if (v4s)
            FL_CUDA(cudaMemcpyAsync(h4, lm->lp.misc.p, sizeof(unsigned long long) * 5, cudaMemcpyDeviceToHost, s));
        const bool sharded_sys = (res->what & FL_OUT_SYSTEM) && res->n != res->m;
        if (sharded_sys) {  // free nodes before / through the range
            const int32_t* fr = res->fidx.as<int32_t>() + (size_t)res->m + 1;
            FL_CUDA(cudaMemcpyAsync(&hn[3], fr + res->col_begin, sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, s));
            FL_CUDA(cudaMemcpyAsync(&hn[4], fr + res->col_begin + res->n, sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, s));
        }
        if ((res->what & FL_OUT_STIFFNESS) && res->arr[FL_A_COL_PTR].p)
            FL_CUDA(cudaMemcpyAsync(&hn[0], res->arr[FL_A_COL_PTR].as<int32_t>() + res->n,
                                    sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        bool replanned = false;
        if (v4s) {
            lm->lp.nnz_bound = (int64_t)h4[0];
            lm->lp.max_inc = (int32_t)h4[1];
            lm->lp.ok = lm->lp.max_inc <= v4_lanes(lm->dim);
            lm->lp.stale = false;
            replanned = true;
            if ((uint32_t)(h4[4] >> 32) & DERR_INDEX) h[CNT_ERR] |= DERR_INDEX;
            // the bucketed fill dropped entries of an over-full bucket
            if ((uint32_t)(h4[4] >> 32) & DERR_V2_OVERFLOW) h[CNT_ERR] |= DERR_V2_OVERFLOW;
        }
        if (lm && lm->stats_stale && !res->v4_used) {  // an asynchronous re-plan ran with the old bounds
            lm->nnz_bound = (int64_t)hst[0];
            lm->max_inc = (int32_t)hst[1];
            lm->stats_stale = false;
            replanned = true;
            if ((uint32_t)(hst[3] & 0xFFFFFFFFull) & DERR_INDEX) h[CNT_ERR] |= DERR_INDEX;
        }
        // a new topology that outgrew the old bounds: redo the column pass sized
        // by the fresh plan (general kernel)
        if (((h[CNT_ERR] & DERR_V2_OVERFLOW) || (replanned && (h[CNT_ERR] & DERR_CAPACITY))) &&
            x->last_valid && !(h[CNT_ERR] & DERR_INDEX)) {
            FL_TRY(rerun_general(res, x));
            FL_CUDA(cudaMemcpyAsync(h, res->counters.p, sizeof(uint32_t) * CNT_WORDS,
                                    cudaMemcpyDeviceToHost, s));
            if ((res->what & FL_OUT_STIFFNESS) && res->arr[FL_A_COL_PTR].p)
                FL_CUDA(cudaMemcpyAsync(&hn[0], res->arr[FL_A_COL_PTR].as<int32_t>() + res->n,
                                        sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            FL_CUDA(cudaStreamSynchronize(s));
        }
        fl_sizes z{};
        z.n = res->n;
        z.nnz = hn[0];
        const uint32_t e = h[CNT_ERR];
        z.n_dir_faces = (int32_t)h[CNT_DIR_FACES];
        z.n_neu_faces = (int32_t)h[CNT_NEU_FACES];
        if (res->what & FL_OUT_PARTITION) {
            z.n_dir = (int32_t)h[CNT_N_DIR];
            z.n_free = res->m - z.n_dir;
            z.n_free_cols = sharded_sys ? hn[4] - hn[3] : z.n_free;
        }
        if (ctx->profile && ctx->timing_pending) {
            float a = 0, b = 0, c = 0;
            cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
            cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
            cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
            ctx->timings[0] = ctx->plan_timed ? a : 0.0;
            ctx->timings[1] = b;
            ctx->timings[2] = c;
            ctx->timings[3] = a + b + c;
            ctx->ktimings[0] = ctx->ktimings[1] = ctx->ktimings[2] = 0.0;
            if (ctx->kernel_timed) {
                float e = 0, f = 0, g = 0;
                cudaEventElapsedTime(&e, ctx->ev[5], ctx->ev[6]);
                cudaEventElapsedTime(&f, ctx->ev[6], ctx->ev[7]);
                cudaEventElapsedTime(&g, ctx->ev[7], ctx->ev[3]);
                ctx->ktimings[0] = e;
                ctx->ktimings[1] = f;
                ctx->ktimings[2] = g;
            }
            ctx->timing_pending = false;
        }
        if (e & DERR_INDEX) return set_error(FL_E_INDEX_OUT_OF_RANGE, "element vertex index out of range");
        if (e & DERR_FLAG) return set_error(FL_E_INVALID_FLAG_VALUE, "boundary flag not in {0,1,2,3}");
        if ((res->what & FL_OUT_PARTITION) && (e & DERR_ROBIN))
            return set_error(FL_E_UNSUPPORTED_BOUNDARY_TYPE,
                             "Robin boundary (flag 3) is not supported");
        if (e & DERR_DEGENERATE) return set_error(FL_E_DEGENERATE_ELEMENT, "degenerate element");
        if (e & DERR_OVERFLOW)
            return set_error(FL_ERR_UNSUPPORTED, "a node has too many incident elements for the column kernel");
        if (e & DERR_CAPACITY) return set_error(FL_ERR_UNSUPPORTED, "internal: output capacity exceeded");
        if (res->what & FL_OUT_SYSTEM) {
            if (z.n_dir_faces == 0)
                return set_error(FL_E_NO_DIRICHLET_BOUNDARY,
                                 "mesh has no Dirichlet faces; use the pure-Neumann path");
            if (x->g_missing)
                return set_error(FL_E_INVALID_PARAMETER,
                                 "mesh has Dirichlet faces but no g_dirichlet was given");
            int32_t* hf = hn + 2;
            FL_CUDA(cudaMemcpyAsync(hf, res->arr[FL_AFF_COL_PTR].as<int32_t>() + z.n_free_cols,
                                    sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            FL_CUDA(cudaStreamSynchronize(s));
            z.nnz_ff = *hf;
        }
        res->sizes = z;
        res->sizes_valid = true;
    }
    *out = res->sizes;
    return FL_OK;
}

static int64_t array_bytes(const fl_result* r, int which) {
    const fl_sizes& z = r->sizes;
    switch (which) {
    case FL_A_COL_PTR: return (r->what & FL_OUT_STIFFNESS) ? 4 * ((int64_t)z.n + 1) : 0;
    case FL_A_ROW_IDX: return (r->what & FL_OUT_STIFFNESS) ? 4 * z.nnz : 0;
    case FL_A_VALUES: return (r->what & FL_OUT_STIFFNESS) ? 8 * z.nnz : 0;
    case FL_B: return (r->what & FL_OUT_LOAD) ? 8 * (int64_t)z.n : 0;
    case FL_U0:
    case FL_B_MOD: return (r->what & (FL_OUT_SYSTEM | kWhatLift)) ? 8 * (int64_t)z.n : 0;
    case FL_DIR_NODES: return (r->what & FL_OUT_PARTITION) ? 4 * (int64_t)z.n_dir : 0;
    case FL_FREE_NODES: return (r->what & FL_OUT_PARTITION) ? 4 * (int64_t)z.n_free : 0;
    case FL_AFF_COL_PTR: return (r->what & FL_OUT_SYSTEM) ? 4 * ((int64_t)z.n_free_cols + 1) : 0;
    case FL_AFF_ROW_IDX: return (r->what & FL_OUT_SYSTEM) ? 4 * z.nnz_ff : 0;
    case FL_AFF_VALUES: return (r->what & FL_OUT_SYSTEM) ? 8 * z.nnz_ff : 0;
    case FL_B_F: return (r->what & FL_OUT_SYSTEM) ? 8 * (int64_t)z.n_free_cols : 0;
    case FL_DIR_FACES: return (r->what & FL_OUT_PARTITION) ? 4 * (int64_t)z.n_dir_faces * r->dim : 0;
    case FL_DIR_FACE_ELEM:
    case FL_DIR_FACE_LOCAL: return (r->what & FL_OUT_PARTITION) ? 4 * (int64_t)z.n_dir_faces : 0;
    case FL_NEU_FACES: return (r->what & FL_OUT_PARTITION) ? 4 * (int64_t)z.n_neu_faces * r->dim : 0;
    case FL_NEU_FACE_ELEM:
    case FL_NEU_FACE_LOCAL: return (r->what & FL_OUT_PARTITION) ? 4 * (int64_t)z.n_neu_faces : 0;
    }
    return -1;
}

FL_API int fl_result_counts_async(fl_result* res, int64_t* dev_out) {
    if (!res || !dev_out || !res->ctx) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (!(res->what & (FL_OUT_STIFFNESS | FL_OUT_LOAD)))
        return set_error(FL_ERR_ARGUMENT, "result holds no assembly");
    FL_CUDA(cudaSetDevice(res->ctx->device));
    return launch_result_counts(res->ctx, res, dev_out);
}

FL_API int fl_result_device_ptr(fl_result* res, int which, const void** ptr, int64_t* bytes) {
    if (!res || !ptr || which < 0 || which >= FL_NUM_ARRAYS)
        return set_error(FL_ERR_ARGUMENT, "bad argument");
    fl_sizes z;
    FL_TRY(fl_result_sizes(res, &z));
    *ptr = res->arr[which].p;
    if (bytes) *bytes = array_bytes(res, which);
    return FL_OK;
}

FL_API int fl_result_copy(fl_result* res, int which, void* dst, int64_t capacity_bytes, int mem) {
    if (!res || which < 0 || which >= FL_NUM_ARRAYS) return set_error(FL_ERR_ARGUMENT, "bad argument");
    fl_sizes z;
    FL_TRY(fl_result_sizes(res, &z));
    const int64_t nb = array_bytes(res, which);
    if (nb > capacity_bytes) return set_error(FL_E_SHAPE_MISMATCH, "destination too small");
    if (nb <= 0) return FL_OK;
    if (!dst) return set_error(FL_ERR_ARGUMENT, "dst is null");
    FL_CUDA(cudaMemcpyAsync(dst, res->arr[which].p, (size_t)nb,
                            mem == FL_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            res->ctx->stream));
    if (mem != FL_MEM_DEVICE) FL_CUDA(cudaStreamSynchronize(res->ctx->stream));
    return FL_OK;
}

FL_API int fl_submatrix(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr,
                        const int32_t* row_idx, const double* values, int32_t n_rows,
                        const int32_t* rows, int32_t n_cols, const int32_t* cols, int mem,
                        fl_result* res) {
    if (!ctx || !res || !col_ptr) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (m < 0 || n < 0 || n_rows < 0 || n_cols < 0) return set_error(FL_E_SHAPE_MISMATCH, "negative size");
    FL_CUDA(cudaSetDevice(ctx->device));
    fl_result_ext* x = ext_of(res);
    auto& st = x->stage.sub;
    const int32_t* d_cp = col_ptr;
    const int32_t* d_ri = row_idx;
    const double* d_va = values;
    const int32_t* d_rows = rows;
    const int32_t* d_cols = cols;
    if (mem != FL_MEM_DEVICE) {
        const int64_t nnz = col_ptr[n];
        FL_TRY(copy_in(ctx, st[0], col_ptr, sizeof(int32_t) * ((size_t)n + 1), FL_MEM_HOST));
        FL_TRY(copy_in(ctx, st[1], row_idx, sizeof(int32_t) * (size_t)nnz, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, st[2], values, sizeof(double) * (size_t)nnz, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, st[3], rows, sizeof(int32_t) * (size_t)n_rows, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, st[4], cols, sizeof(int32_t) * (size_t)n_cols, FL_MEM_HOST));
        d_cp = st[0].as<int32_t>();
        d_ri = st[1].as<int32_t>();
        d_va = st[2].as<double>();
        d_rows = st[3].as<int32_t>();
        d_cols = st[4].as<int32_t>();
    }
    FL_TRY(res->fidx.ensure(sizeof(int32_t) * ((size_t)m + 1 + (size_t)n_cols + 1)));
    int32_t* row_map = res->fidx.as<int32_t>();
    int32_t* cnt = row_map + m + 1;
    uint32_t* d_err = res->counters.as<uint32_t>();
    FL_CUDA(cudaMemsetAsync(d_err, 0, sizeof(uint32_t) * CNT_WORDS, ctx->stream));
    int64_t nnz = 0;
    FL_TRY(launch_submatrix(ctx, m, n, d_cp, d_ri, d_va, n_rows, d_rows, n_cols, d_cols, res,
                            row_map, cnt, d_err, &nnz));
    res->what = FL_OUT_STIFFNESS;
    res->n = n_cols;
    res->m = n_rows;
    res->col_begin = 0;
    res->sizes = fl_sizes{};
    res->sizes.n = n_cols;
    res->sizes.nnz = nnz;
    res->sizes_valid = true;
    return FL_OK;
}

// ---- solve -----------------------------------------------------
static int cg_check(const fl_cg_options* o) {
    if (!o) return set_error(FL_ERR_ARGUMENT, "null options");
    if (!(o->rel_tol > 0.0)) return set_error(FL_E_INVALID_PARAMETER, "rel_tol must be positive");
    return FL_OK;
}

FL_API int fl_cg_solve(fl_ctx* ctx, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                       const double* values, const double* b, int mem, const fl_cg_options* opts,
                       double* x, int64_t* iterations, double* relres, int32_t* converged) {
    if (!ctx || !col_ptr || !x || !iterations || !relres || !converged || (n > 0 && !b))
        return set_error(FL_ERR_ARGUMENT, "null argument");
    if (n < 0) return set_error(FL_E_SHAPE_MISMATCH, "cg_solve: negative size");
    FL_TRY(cg_check(opts));
    FL_CUDA(cudaSetDevice(ctx->device));
    if (mem == FL_MEM_DEVICE)
        return cg_solve_device(ctx, n, col_ptr, row_idx, values, b, opts->rel_tol, opts->max_iter,
                               opts->preconditioner, x, iterations, relres, converged);
    // host arrays: stage on the device
    DevBuf dcp, dri, dva, db, dx;
    auto release = [&]() {
        dcp.release();
        dri.release();
        dva.release();
        db.release();
        dx.release();
    };
    int rc = copy_in(ctx, dcp, col_ptr, sizeof(int32_t) * ((size_t)n + 1), FL_MEM_HOST);
    const int64_t nnz = n >= 0 ? col_ptr[n] : 0;
    if (!rc) rc = copy_in(ctx, dri, row_idx, sizeof(int32_t) * (size_t)nnz, FL_MEM_HOST);
    if (!rc) rc = copy_in(ctx, dva, values, sizeof(double) * (size_t)nnz, FL_MEM_HOST);
    if (!rc) rc = copy_in(ctx, db, b, sizeof(double) * (size_t)n, FL_MEM_HOST);
    if (!rc) rc = dx.ensure(sizeof(double) * (size_t)std::max(n, 1));
    if (!rc)
        rc = cg_solve_device(ctx, n, dcp.as<int32_t>(), dri.as<int32_t>(), dva.as<double>(),
                             db.as<double>(), opts->rel_tol, opts->max_iter, opts->preconditioner,
                             dx.as<double>(), iterations, relres, converged);
    if (!rc && n > 0) {
        cudaError_t e = cudaMemcpyAsync(x, dx.p, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost,
                                        ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
    }
    cudaStreamSynchronize(ctx->stream);
    release();
    return rc;
}

FL_API int fl_from_triplets(fl_ctx* ctx, int32_t m, int32_t n, int64_t count, const int32_t* ii,
                            const int32_t* jj, const double* ss, int mem, fl_result* res) {
    if (!ctx || !res || (count > 0 && (!ii || !jj || !ss))) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (m < 0 || n < 0) return set_error(FL_E_SHAPE_MISMATCH, "negative matrix dimension");
    if (count < 0 || count >= ((int64_t)1 << 31))
        return set_error(FL_ERR_UNSUPPORTED, "triplet count outside [0, 2^31)");
    FL_CUDA(cudaSetDevice(ctx->device));
    fl_result_ext* x = ext_of(res);
    x->last_valid = false;
    const int32_t *di = ii, *dj = jj;
    const double* ds = ss;
    if (mem != FL_MEM_DEVICE) {
        FL_TRY(copy_in(ctx, x->stage.sub[0], ii, sizeof(int32_t) * (size_t)count, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, x->stage.sub[1], jj, sizeof(int32_t) * (size_t)count, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, x->stage.sub[2], ss, sizeof(double) * (size_t)count, FL_MEM_HOST));
        di = x->stage.sub[0].as<int32_t>();
        dj = x->stage.sub[1].as<int32_t>();
        ds = x->stage.sub[2].as<double>();
    }
    return launch_from_triplets(ctx, m, n, count, di, dj, ds, res);
}

FL_API int fl_apply_dirichlet(fl_ctx* ctx, fl_mesh* mesh, int32_t m, int32_t n, const int32_t* col_ptr,
                              const int32_t* row_idx, const double* values, int64_t b_len, const double* b,
                              int mem, const fl_field* g, fl_result* res) {
    if (!ctx || !mesh || !res || !col_ptr) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (!field_ok(g)) return set_error(FL_ERR_ARGUMENT, "invalid field descriptor");
    FL_CUDA(cudaSetDevice(ctx->device));
    if (mesh->col_begin != 0 || mesh->col_end != mesh->n_nodes)
        return set_error(FL_ERR_UNSUPPORTED, "fl_apply_dirichlet needs the whole mesh (no column range)");
    const cudaStream_t s = ctx->stream;
    const int32_t N = mesh->n_nodes;
    fl_result_ext* x = ext_of(res);
    x->last_valid = false;
    res->sizes_valid = false;
    res->v4_used = false;
    res->what = FL_OUT_PARTITION;
    res->n = N;
    res->m = N;
    res->col_begin = 0;
    res->dim = mesh->dim;
    // partition_boundary first (system.hpp:185): Robin flags, then no Dirichlet faces
    uint32_t* counters = res->counters.as<uint32_t>();
    FL_CUDA(cudaMemsetAsync(counters, 0, sizeof(uint32_t) * CNT_WORDS, s));
    const size_t n1 = (size_t)N + 1;
    FL_TRY(res->is_dir.ensure(n1));
    FL_TRY(res->is_neu.ensure(n1));
    FL_TRY(res->fidx.ensure(sizeof(int32_t) * 2 * n1));
    FL_TRY(res->arr[FL_DIR_NODES].ensure(sizeof(int32_t) * n1));
    FL_TRY(res->arr[FL_FREE_NODES].ensure(sizeof(int32_t) * n1));
    FL_TRY(launch_partition(ctx, mesh, res));
    FL_TRY(launch_face_lists(ctx, mesh, res));
    uint32_t* h = static_cast<uint32_t*>(ctx->pinned);
    FL_CUDA(cudaMemcpyAsync(h, counters, sizeof(uint32_t) * CNT_WORDS, cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    if (h[CNT_ERR] & DERR_INDEX) return set_error(FL_E_INDEX_OUT_OF_RANGE, "element vertex index out of range");
    if (h[CNT_ERR] & DERR_FLAG) return set_error(FL_E_INVALID_FLAG_VALUE, "boundary flag not in {0,1,2,3}");
    if (h[CNT_ERR] & DERR_ROBIN)
        return set_error(FL_E_UNSUPPORTED_BOUNDARY_TYPE, "Robin boundary (flag 3) is not supported");
    if (h[CNT_DIR_FACES] == 0)
        return set_error(FL_E_NO_DIRICHLET_BOUNDARY, "mesh has no Dirichlet faces; use the pure-Neumann path");
    if (m != N || n != N || b_len != N) return set_error(FL_E_SHAPE_MISMATCH, "apply_dirichlet: size mismatch");
    if (N > 0 && (!b || !row_idx || !values)) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (!g || g->kind == FL_FIELD_NONE)  // the reference calls g: an empty std::function throws
        return set_error(FL_ERR_ARGUMENT, "apply_dirichlet: g is empty");
    FieldDesc gd;
    FL_TRY(field_desc(ctx, g, N, x->stage.g_dir, &gd, "g_dirichlet"));
    const int32_t* dcp = col_ptr;
    const int32_t* dri = row_idx;
    const double* dva = values;
    const double* db = b;
    if (mem != FL_MEM_DEVICE) {
        const int64_t nnz = col_ptr[n];
        FL_TRY(copy_in(ctx, x->stage.sub[0], col_ptr, sizeof(int32_t) * ((size_t)n + 1), FL_MEM_HOST));
        FL_TRY(copy_in(ctx, x->stage.sub[1], row_idx, sizeof(int32_t) * (size_t)nnz, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, x->stage.sub[2], values, sizeof(double) * (size_t)nnz, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, x->stage.sub[3], b, sizeof(double) * (size_t)N, FL_MEM_HOST));
        dcp = x->stage.sub[0].as<int32_t>();
        dri = x->stage.sub[1].as<int32_t>();
        dva = x->stage.sub[2].as<double>();
        db = x->stage.sub[3].as<double>();
    }
    FL_TRY(launch_dirichlet_lift(ctx, mesh, res, gd, dcp, dri, dva, db));
    res->what = FL_OUT_PARTITION | kWhatLift;
    return FL_OK;
}

FL_API int fl_accumulate(fl_ctx* ctx, int64_t count, const int32_t* idx, const double* vals, int32_t size,
                         double* out, int mem) {
    if (!ctx || (count > 0 && (!idx || !vals)) || (size > 0 && !out)) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (size < 0 || count < 0) return set_error(FL_E_SHAPE_MISMATCH, "accumulate: negative size");
    FL_CUDA(cudaSetDevice(ctx->device));
    fl_result* col = nullptr;
    FL_TRY(fl_result_create(ctx, &col));
    DevBuf zeros, dout;
    int rc = zeros.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(count, 1));
    if (!rc && count > 0) {
        const cudaError_t e = cudaMemsetAsync(zeros.p, 0, sizeof(int32_t) * (size_t)count, ctx->stream);
        if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
    }
    // the one-column from_triplets of (idx, 0, vals): stable by index, each
    // index's values summed in their original order (sparse.hpp:61-115)
    if (!rc) {
        fl_result_ext* x = ext_of(col);
        const int32_t* di = idx;
        const double* dv = vals;
        if (mem != FL_MEM_DEVICE) {
            rc = copy_in(ctx, x->stage.sub[0], idx, sizeof(int32_t) * (size_t)count, FL_MEM_HOST);
            if (!rc) rc = copy_in(ctx, x->stage.sub[2], vals, sizeof(double) * (size_t)count, FL_MEM_HOST);
            di = x->stage.sub[0].as<int32_t>();
            dv = x->stage.sub[2].as<double>();
        }
        if (!rc) rc = launch_from_triplets(ctx, size, 1, count, di, zeros.as<int32_t>(), dv, col);
    }
    fl_sizes z{};
    if (!rc) rc = fl_result_sizes(col, &z);  // index_out_of_range surfaces here
    double* target = out;
    if (!rc && mem != FL_MEM_DEVICE) {
        rc = dout.ensure(sizeof(double) * (size_t)std::max(size, 1));
        target = dout.as<double>();
    }
    if (!rc && size > 0) rc = launch_scatter_column(ctx, col, size, target);
    if (!rc && mem != FL_MEM_DEVICE && size > 0) {
        const cudaError_t e = cudaMemcpyAsync(out, target, sizeof(double) * (size_t)size, cudaMemcpyDeviceToHost,
                                              ctx->stream);
        if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
    }
    cudaStreamSynchronize(ctx->stream);
    zeros.release();
    dout.release();
    fl_result_destroy(col);
    if (rc == FL_E_INDEX_OUT_OF_RANGE) set_error(rc, "accumulate: index out of range");
    return rc;
}

FL_API int fl_solve_neumann(fl_ctx* ctx, fl_mesh* mesh, fl_result* res, int32_t pin,
                            const fl_cg_options* opts, double* u, int mem, int64_t* iterations,
                            double* relres) {
    if (!ctx || !mesh || !res || !u || !iterations || !relres)
        return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_TRY(cg_check(opts));
    if ((res->what & (FL_OUT_STIFFNESS | FL_OUT_LOAD)) != (FL_OUT_STIFFNESS | FL_OUT_LOAD))
        return set_error(FL_ERR_ARGUMENT, "result needs FL_OUT_STIFFNESS | FL_OUT_LOAD");
    fl_sizes z;
    FL_TRY(fl_result_sizes(res, &z));
    if (z.n != res->m || res->m != mesh->n_nodes)
        return set_error(FL_ERR_UNSUPPORTED, "fl_solve_neumann needs the whole mesh");
    FL_CUDA(cudaSetDevice(ctx->device));
    DevBuf du;
    double* target = u;
    int rc = FL_OK;
    if (mem != FL_MEM_DEVICE) {
        rc = du.ensure(sizeof(double) * (size_t)std::max(z.n, 1));
        target = du.as<double>();
    }
    int32_t conv = 1;
    if (!rc)
        rc = solve_neumann_device(ctx, mesh->dim, z.n, mesh->n_elems, mesh->nodes.as<double>(),
                                  mesh->elems.as<int32_t>(), res->arr[FL_A_COL_PTR].as<int32_t>(),
                                  res->arr[FL_A_ROW_IDX].as<int32_t>(), res->arr[FL_A_VALUES].as<double>(),
                                  res->arr[FL_B].as<double>(), pin, opts->rel_tol, opts->max_iter,
                                  opts->preconditioner, target, iterations, relres, &conv);
    if (!rc && mem != FL_MEM_DEVICE && z.n > 0) {
        cudaError_t e = cudaMemcpy(u, target, sizeof(double) * (size_t)z.n, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
    }
    du.release();
    if (!rc && !conv)
        return set_error(FL_E_MAX_ITER_EXCEEDED, "cg did not reach rel_tol in max_iter iterations");
    return rc;
}

FL_API int fl_matvec(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr,
                     const int32_t* row_idx, const double* values, const double* x, double* y,
                     int mem) {
    if (!ctx || !col_ptr || (m > 0 && !y) || (n > 0 && !x)) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (m < 0 || n < 0) return set_error(FL_E_SHAPE_MISMATCH, "matvec: negative size");
    FL_CUDA(cudaSetDevice(ctx->device));
    if (mem == FL_MEM_DEVICE) return matvec_device(ctx, m, n, col_ptr, row_idx, values, x, y);
    DevBuf dcp, dri, dva, dx, dy;
    const int64_t nnz = col_ptr[n];
    int rc = copy_in(ctx, dcp, col_ptr, sizeof(int32_t) * ((size_t)n + 1), FL_MEM_HOST);
    if (!rc) rc = copy_in(ctx, dri, row_idx, sizeof(int32_t) * (size_t)nnz, FL_MEM_HOST);
    if (!rc) rc = copy_in(ctx, dva, values, sizeof(double) * (size_t)nnz, FL_MEM_HOST);
    if (!rc) rc = copy_in(ctx, dx, x, sizeof(double) * (size_t)n, FL_MEM_HOST);
    if (!rc) rc = dy.ensure(sizeof(double) * (size_t)std::max(m, 1));
    if (!rc) rc = matvec_device(ctx, m, n, dcp.as<int32_t>(), dri.as<int32_t>(), dva.as<double>(),
                                dx.as<double>(), dy.as<double>());
    if (!rc && m > 0) {
        cudaError_t e = cudaMemcpy(y, dy.p, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
    }
    dcp.release();
    dri.release();
    dva.release();
    dx.release();
    dy.release();
    return rc;
}

FL_API int fl_solve_system(fl_ctx* ctx, fl_result* res, const fl_cg_options* opts, double* u,
                           int mem, int64_t* iterations, double* relres) {
    if (!ctx || !res || !u || !iterations || !relres) return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_TRY(cg_check(opts));
    if (!(res->what & FL_OUT_SYSTEM)) return set_error(FL_ERR_ARGUMENT, "result holds no FL_OUT_SYSTEM");
    fl_sizes z;
    FL_TRY(fl_result_sizes(res, &z));
    if (z.n != res->m) return set_error(FL_ERR_UNSUPPORTED, "fl_solve_system needs the whole mesh");
    FL_CUDA(cudaSetDevice(ctx->device));
    DevBuf dx, du;
    int32_t conv = 1;
    int rc = dx.ensure(sizeof(double) * (size_t)std::max(z.n_free, 1));
    if (!rc)
        rc = cg_solve_device(ctx, z.n_free, res->arr[FL_AFF_COL_PTR].as<int32_t>(),
                             res->arr[FL_AFF_ROW_IDX].as<int32_t>(), res->arr[FL_AFF_VALUES].as<double>(),
                             res->arr[FL_B_F].as<double>(), opts->rel_tol, opts->max_iter,
                             opts->preconditioner, dx.as<double>(), iterations, relres, &conv);
    double* target = u;
    if (!rc && mem != FL_MEM_DEVICE) {
        rc = du.ensure(sizeof(double) * (size_t)std::max(z.n, 1));
        target = du.as<double>();
    }
    if (!rc && z.n > 0) {
        cudaError_t e = cudaMemcpyAsync(target, res->arr[FL_U0].p, sizeof(double) * (size_t)z.n,
                                        cudaMemcpyDeviceToDevice, ctx->stream);
        if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
        if (!rc) rc = scatter_free(ctx, z.n_free, res->arr[FL_FREE_NODES].as<int32_t>(), dx.as<double>(), target);
        if (!rc && mem != FL_MEM_DEVICE) {
            e = cudaMemcpyAsync(u, target, sizeof(double) * (size_t)z.n, cudaMemcpyDeviceToHost, ctx->stream);
            if (e != cudaSuccess) rc = set_error(FL_ERR_CUDA, cudaGetErrorString(e));
        }
    }
    cudaStreamSynchronize(ctx->stream);
    dx.release();
    du.release();
    if (!rc && !conv)
        return set_error(FL_E_MAX_ITER_EXCEEDED, "cg did not reach rel_tol in max_iter iterations");
    return rc;
}

FL_API int fl_phase_cycles(fl_ctx* ctx, uint64_t* out6) {
    if (!ctx || !out6) return set_error(FL_ERR_ARGUMENT, "null argument");
    for (int i = 0; i < 6; ++i) out6[i] = 0;
    if (!ctx->phase_timing) return FL_OK;
    FL_CUDA(cudaMemcpyAsync(ctx->pinned, ctx->phases.p, sizeof(unsigned long long) * 6,
                            cudaMemcpyDeviceToHost, ctx->stream));
    FL_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 6; ++i) out6[i] = static_cast<const unsigned long long*>(ctx->pinned)[i];
    return FL_OK;
}

FL_API int fl_selftest_div(fl_ctx* ctx, int64_t n, const double* a, const double* b,
                           double* q_fast, double* q_ieee, int mem) {
    if (!ctx) return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_CUDA(cudaSetDevice(ctx->device));
    DevBuf da, db, dq, di;
    const double *pa = a, *pb = b;
    double *pq = q_fast, *pi = q_ieee;
    const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
    if (mem != FL_MEM_DEVICE) {
        FL_TRY(copy_in(ctx, da, a, sizeof(double) * (size_t)n, FL_MEM_HOST));
        FL_TRY(copy_in(ctx, db, b, sizeof(double) * (size_t)n, FL_MEM_HOST));
        FL_TRY(dq.ensure(bytes));
        FL_TRY(di.ensure(bytes));
        pa = da.as<double>();
        pb = db.as<double>();
        pq = dq.as<double>();
        pi = di.as<double>();
    }
    int rc = launch_selftest_div(ctx, n, pa, pb, pq, pi);
    if (!rc && mem != FL_MEM_DEVICE && n > 0) {
        cudaMemcpyAsync(q_fast, pq, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(q_ieee, pi, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream);
    }
    cudaStreamSynchronize(ctx->stream);
    da.release();
    db.release();
    dq.release();
    di.release();
    return rc;
}

static double host_field(int kind, double value, double x, double y, double z) {
    const double pi = 3.14159265358979323846;  // std::numbers::pi
    switch (kind) {
    case FL_FIELD_CONST: return value;
    case FL_FIELD_X: return x;
    case FL_FIELD_XYZ: return x + y + z;
    case FL_FIELD_SINSIN: return std::sin(pi * x) * std::sin(pi * y);
    }
    return 0.0;
}

// Cartesian point q of element t under `rule` (the reference's formulas)
static void host_point(int rule, int dim, const double* nodes, const int32_t* v, int q, double x[3]) {
    static const int tri[3][2] = {{1, 2}, {2, 0}, {0, 1}};
    static const int tet[4][3] = {{1, 3, 2}, {0, 2, 3}, {0, 3, 1}, {0, 1, 2}};
    auto P = [&](int32_t k, int c) { return c < dim ? nodes[(size_t)k * dim + c] : 0.0; };
    x[0] = x[1] = x[2] = 0.0;
    if (rule == 0 && dim == 2) {  // system.hpp:86-90
        for (int c = 0; c < 2; ++c) x[c] = (P(v[tri[q][0]], c) + P(v[tri[q][1]], c)) / 2.0;
    } else if (rule == 0) {  // system.hpp:103-107
        for (int k = 0; k < 4; ++k) {
            const double lam = (k == q) ? 0.58541019662496845 : 0.13819660112501051;
            for (int c = 0; c < 3; ++c) x[c] += lam * P(v[k], c);
        }
    } else if (dim == 2) {  // system.hpp:143
        for (int c = 0; c < 2; ++c) x[c] = (P(v[tri[q][0]], c) + P(v[tri[q][1]], c)) / 2.0;
    } else {  // system.hpp:160-161
        for (int c = 0; c < 3; ++c)
            x[c] = (P(v[tet[q][0]], c) + P(v[tet[q][1]], c) + P(v[tet[q][2]], c)) / 3.0;
    }
}

FL_API int fl_host_sample(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, int rule, int kind, double value, double* out) {
    if ((dim != 2 && dim != 3) || !out || (n_nodes > 0 && !nodes) || (n_elems > 0 && !elems) ||
        rule < 0 || rule > 3)
        return set_error(FL_ERR_ARGUMENT, "bad argument");
    const int nv = dim + 1;
    auto P = [&](int32_t k, int c) { return c < dim ? nodes[(size_t)k * dim + c] : 0.0; };
    if (rule == 2) {
        for (int32_t k = 0; k < n_nodes; ++k) out[k] = host_field(kind, value, P(k, 0), P(k, 1), P(k, 2));
        return FL_OK;
    }
    for (int32_t t = 0; t < n_elems; ++t) {
        const int32_t* v = elems + (size_t)t * nv;
        if (rule == 1) {  // SURVEY.md §8 a11 barycentre (first coordinate)
            double xs = P(v[0], 0);
            for (int k = 1; k < nv; ++k) xs = xs + P(v[k], 0);
            const double xbar = xs / (double)nv;
            out[t] = kind == FL_FIELD_COEF_C5 ? 1.0 + 0.5 * std::sin((2.0 * 3.14159265358979323846) * xbar)
                                              : host_field(kind, value, xbar, 0.0, 0.0);
            continue;
        }
        for (int q = 0; q < nv; ++q) {
            double x[3];
            host_point(rule, dim, nodes, v, q, x);
            out[(size_t)t * nv + q] = host_field(kind, value, x[0], x[1], x[2]);
        }
    }
    return FL_OK;
}

FL_API int fl_host_points(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, int rule, double* xyz) {
    if ((dim != 2 && dim != 3) || !xyz || (n_nodes > 0 && !nodes) || (n_elems > 0 && !elems) ||
        (rule != 0 && rule != 3))
        return set_error(FL_ERR_ARGUMENT, "bad argument");
    const int nv = dim + 1;
    for (int32_t t = 0; t < n_elems; ++t)
        for (int q = 0; q < nv; ++q) host_point(rule, dim, nodes, elems + (size_t)t * nv, q, xyz + ((size_t)t * nv + q) * 3);
    return FL_OK;
}

}  // extern "C"
