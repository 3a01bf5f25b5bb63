/* nccl_shim.c -- TEST INFRASTRUCTURE: a host-staged implementation of the dozen NCCL entry
 * points the library's multi-GPU transport resolves at run time (paper_1408_4599_b200/csrc/
 * nccl_api.hpp), for p processes that share ONE GPU.  NCCL itself refuses two ranks of a
 * communicator on one device, so on a one-GPU box the library's NCCL code path -- grouped
 * send/recv of the halo and migration records, the all-gather of the record counts, the
 * all-reduces of cell loads, observables and failure flags -- can only execute through a
 * stand-in with NCCL's calling convention.  The library loads it when MARDYN_NCCL_LIB names
 * it (tests/test_gpu_nccl_shim.py).
 *
 * Semantics kept from NCCL: point-to-point operations between a pair of ranks match in
 * issue order; operations between ncclGroupStart / ncclGroupEnd are issued together (all
 * sends first, then all receives, so a group never deadlocks); collectives are ordered per
 * communicator; every operation is ordered after the work already on its stream.  What
 * differs: each operation is completed on the host before the call returns (stream
 * synchronised, device -> host copy, a file in a shared directory, host -> device copy), so
 * nothing is left in flight and nothing here can run under CUDA stream capture.  No GPU
 * kernel waits on another process (the one-GPU rule of the profiling guide).
 *
 * Transport: files <dir>/p<src>_<dst>_<seq> (read once, then removed by the receiver) and
 * <dir>/c<seq>_<rank> (a rank removes its own collective file two collectives later: by then
 * every rank has read it).  Files appear atomically (write + rename).  MDSHIM_HOST=1 treats
 * every buffer as host memory (no CUDA at all: the CPU test of the shim's own semantics). */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <errno.h>
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <unistd.h>

#define MAXR 64
#define MAXOPS 4096

struct ncclComm {
    int rank, nranks;
    char dir[NCCL_UNIQUE_ID_BYTES];
    uint64_t sseq[MAXR], rseq[MAXR], cseq;
};

/* ---- device access through the driver API (the process's current context) */
typedef int (*pSync)(void*);
typedef int (*pD2H)(void*, unsigned long long, size_t);
typedef int (*pH2D)(unsigned long long, const void*, size_t, void*);
static pSync cu_sync;
static pD2H cu_d2h;
static pH2D cu_h2d;
static int host_mode = -1;
static FILE* logf;

/* MDSHIM_LOG=<dir>: one line per operation in <dir>/shim_rank<r>.log (debugging aid) */
static void logop(const struct ncclComm* c, const char* what, int peer, unsigned long long seq, size_t bytes, int rc)
{
    if (!logf) {
        const char* d = getenv("MDSHIM_LOG");
        if (!d) return;
        char path[512];
        snprintf(path, sizeof path, "%s/shim_rank%d.log", d, c->rank);
        logf = fopen(path, "w");
        if (!logf) return;
    }
    fprintf(logf, "%s peer %d seq %llu bytes %zu rc %d\n", what, peer, seq, bytes, rc);
    fflush(logf);
}

static int cu_init(void)
{
    if (host_mode < 0) {
        const char* e = getenv("MDSHIM_HOST");
        host_mode = e && e[0] == '1';
    }
    if (host_mode || cu_sync) return 0;
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) return -1;
    cu_sync = (pSync)dlsym(h, "cuStreamSynchronize");
    cu_d2h = (pD2H)dlsym(h, "cuMemcpyDtoH_v2");
    cu_h2d = (pH2D)dlsym(h, "cuMemcpyHtoDAsync_v2");
    return cu_sync && cu_d2h && cu_h2d ? 0 : -1;
}
static int to_host(void* dst, const void* src, size_t n, cudaStream_t s)
{
    if (host_mode) { memcpy(dst, src, n); return 0; }
    if (cu_sync((void*)s)) return -1;
    return n ? cu_d2h(dst, (unsigned long long)(uintptr_t)src, n) : 0;
}
/* on the operation's stream, then synchronised: a synchronous cuMemcpyHtoD from pageable
 * memory may return before the data reaches the device, and the library reads the result
 * on its own (non-blocking) stream */
static int to_dev(void* dst, const void* src, size_t n, cudaStream_t s)
{
    if (host_mode) { memcpy(dst, src, n); return 0; }
    if (!n) return 0;
    const int e = cu_h2d((unsigned long long)(uintptr_t)dst, src, n, (void*)s);
    return e ? e : cu_sync((void*)s);
}

static size_t tsize(ncclDataType_t t)
{
    switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
    }
}

/* ---- files */
static int put_file(const char* path, const void* buf, size_t n)
{
    char tmp[512];
    snprintf(tmp, sizeof tmp, "%s.tmp", path);
    FILE* f = fopen(tmp, "wb");
    if (!f) return -1;
    if (n && fwrite(buf, 1, n, f) != n) { fclose(f); return -1; }
    if (fclose(f)) return -1;
    return rename(tmp, path);
}
static int get_file(const char* path, void* buf, size_t n, int remove_after)
{
    const char* to = getenv("MDSHIM_TIMEOUT_S");
    const double limit = to ? atof(to) : 300.0;
    double waited = 0.0;
    struct stat st;
    while (stat(path, &st) != 0) {
        usleep(100);
        waited += 1e-4;
        if (waited > limit) return -2;
    }
    if ((size_t)st.st_size != n) return -3;      /* size mismatch: mismatched send / recv */
    FILE* f = fopen(path, "rb");
    if (!f) return -1;
    const size_t got = n ? fread(buf, 1, n, f) : 0;
    fclose(f);
    if (got != n) return -1;
    if (remove_after) unlink(path);
    return 0;
}

/* ---- API */
const char* ncclGetErrorString(ncclResult_t r)
{
    return r == ncclSuccess ? "no error" : "nccl_shim: operation failed (file transport)";
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id)
{
    const char* base = getenv("MDSHIM_DIR");
    char tmpl[NCCL_UNIQUE_ID_BYTES];
    snprintf(tmpl, sizeof tmpl, "%s/mdshim_XXXXXX", base ? base : "/tmp");
    if (!mkdtemp(tmpl)) return ncclSystemError;
    memset(id, 0, sizeof *id);
    memcpy(id->internal, tmpl, strlen(tmpl));
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank)
{
    if (nranks < 1 || nranks > MAXR || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    if (cu_init()) return ncclSystemError;
    struct ncclComm* c = (struct ncclComm*)calloc(1, sizeof *c);
    if (!c) return ncclSystemError;
    c->rank = rank;
    c->nranks = nranks;
    memcpy(c->dir, id.internal, NCCL_UNIQUE_ID_BYTES - 1);
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) { free(c); return ncclSuccess; }
ncclResult_t ncclCommAbort(ncclComm_t c) { free(c); return ncclSuccess; }
ncclResult_t ncclCommGetAsyncError(ncclComm_t c, ncclResult_t* e) { (void)c; *e = ncclSuccess; return ncclSuccess; }

typedef struct {
    int send;
    void* buf;
    size_t bytes;
    int peer;
    ncclComm_t comm;
    cudaStream_t stream;
} Op;
static __thread Op ops[MAXOPS];
static __thread int nops, depth;

static ncclResult_t do_send(const Op* o)
{
    ncclComm_t c = o->comm;
    void* h = malloc(o->bytes ? o->bytes : 1);
    if (!h) return ncclSystemError;
    char path[512];
    const unsigned long long q = c->sseq[o->peer]++;
    snprintf(path, sizeof path, "%s/p%d_%d_%llu", c->dir, c->rank, o->peer, q);
    int e = to_host(h, o->buf, o->bytes, o->stream);
    if (!e) e = put_file(path, h, o->bytes);
    free(h);
    logop(c, "send", o->peer, q, o->bytes, e);
    return e ? ncclSystemError : ncclSuccess;
}

static ncclResult_t do_recv(const Op* o)
{
    ncclComm_t c = o->comm;
    void* h = malloc(o->bytes ? o->bytes : 1);
    if (!h) return ncclSystemError;
    char path[512];
    const unsigned long long q = c->rseq[o->peer]++;
    snprintf(path, sizeof path, "%s/p%d_%d_%llu", c->dir, o->peer, c->rank, q);
    int e = host_mode ? 0 : cu_sync((void*)o->stream);     /* earlier work on the stream first */
    if (e) e = 1000 + e;
    if (!e) e = get_file(path, h, o->bytes, 1);
    if (!e) e = to_dev(o->buf, h, o->bytes, o->stream);
    free(h);
    logop(c, "recv", o->peer, q, o->bytes, e);
    return e ? (e == -3 ? ncclInvalidUsage : ncclSystemError) : ncclSuccess;
}

static ncclResult_t flush_group(void)
{
    ncclResult_t r = ncclSuccess;
    for (int i = 0; i < nops && r == ncclSuccess; ++i)
        if (ops[i].send) r = do_send(&ops[i]);
    for (int i = 0; i < nops && r == ncclSuccess; ++i)
        if (!ops[i].send) r = do_recv(&ops[i]);
    nops = 0;
    return r;
}

ncclResult_t ncclGroupStart(void) { ++depth; return ncclSuccess; }
ncclResult_t ncclGroupEnd(void)
{
    if (depth <= 0) return ncclInvalidUsage;
    if (--depth == 0) return flush_group();
    return ncclSuccess;
}

static ncclResult_t p2p(int send, const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c,
                        cudaStream_t s)
{
    if (!c || peer < 0 || peer >= c->nranks) return ncclInvalidArgument;
    if (nops == MAXOPS) return ncclInternalError;
    ops[nops++] = (Op){send, (void*)buf, count * tsize(t), peer, c, s};
    return depth == 0 ? flush_group() : ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s)
{
    return p2p(1, buf, count, t, peer, c, s);
}
ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s)
{
    return p2p(0, buf, count, t, peer, c, s);
}

/* every rank's contribution of a collective, in rank order */
static ncclResult_t exchange_all(ncclComm_t c, const void* dev, size_t bytes, cudaStream_t s, char* all)
{
    if (depth > 0) return ncclInvalidUsage;      /* collectives inside a group: not used by the library */
    const uint64_t q = c->cseq++;
    char path[512];
    if (q >= 2) {
        snprintf(path, sizeof path, "%s/c%llu_%d", c->dir, (unsigned long long)(q - 2), c->rank);
        unlink(path);
    }
    char* mine = all + (size_t)c->rank * bytes;
    const int eh = to_host(mine, dev, bytes, s);
    logop(c, "coll", -1, q, bytes, eh);
    if (eh) return ncclSystemError;
    snprintf(path, sizeof path, "%s/c%llu_%d", c->dir, (unsigned long long)q, c->rank);
    if (put_file(path, mine, bytes)) return ncclSystemError;
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        snprintf(path, sizeof path, "%s/c%llu_%d", c->dir, (unsigned long long)q, r);
        const int e = get_file(path, all + (size_t)r * bytes, bytes, 0);
        if (e) {
            logop(c, "coll-fail", r, q, bytes, e);
            return e == -3 ? ncclInvalidUsage : ncclSystemError;
        }
    }
    return ncclSuccess;
}

#define REDUCE(T)                                                                               \
    for (size_t i = 0; i < count; ++i) {                                                        \
        T acc = ((const T*)all)[i];                                                             \
        for (int r = 1; r < c->nranks; ++r) {                                                   \
            const T v = ((const T*)(all + (size_t)r * bytes))[i];                               \
            acc = op == ncclSum ? acc + v : op == ncclProd ? acc * v : op == ncclMax ? (v > acc ? v : acc) \
                                                                                       : (v < acc ? v : acc); \
        }                                                                                       \
        ((T*)out)[i] = acc;                                                                     \
    }

ncclResult_t ncclAllReduce(const void* sb, void* rb, size_t count, ncclDataType_t t, ncclRedOp_t op, ncclComm_t c,
                           cudaStream_t s)
{
    if (op != ncclSum && op != ncclProd && op != ncclMax && op != ncclMin) return ncclInvalidArgument;
    const size_t bytes = count * tsize(t);
    char* all = (char*)malloc((size_t)c->nranks * bytes + 1);
    char* out = (char*)malloc(bytes + 1);
    if (!all || !out) { free(all); free(out); return ncclSystemError; }
    ncclResult_t r = exchange_all(c, sb, bytes, s, all);
    if (r == ncclSuccess) {
        switch (t) {          /* rank order, as NCCL's ring would not promise: exact for integers */
        case ncclInt32: REDUCE(int32_t) break;
        case ncclUint32: REDUCE(uint32_t) break;
        case ncclInt64: REDUCE(int64_t) break;
        case ncclUint64: REDUCE(uint64_t) break;
        case ncclFloat32: REDUCE(float) break;
        case ncclFloat64: REDUCE(double) break;
        default: r = ncclInvalidArgument;
        }
    }
    if (r == ncclSuccess && to_dev(rb, out, bytes, s)) r = ncclSystemError;
    free(all);
    free(out);
    return r;
}

ncclResult_t ncclAllGather(const void* sb, void* rb, size_t count, ncclDataType_t t, ncclComm_t c, cudaStream_t s)
{
    const size_t bytes = count * tsize(t);
    char* all = (char*)malloc((size_t)c->nranks * bytes + 1);
    if (!all) return ncclSystemError;
    ncclResult_t r = exchange_all(c, sb, bytes, s, all);
    if (logf && t == ncclInt64 && c->nranks * count <= 64) {
        fprintf(logf, "allgather int64:");
        for (size_t i = 0; i < c->nranks * count; ++i) fprintf(logf, " %lld", (long long)((int64_t*)all)[i]);
        fprintf(logf, "\n");
    }
    if (r == ncclSuccess && to_dev(rb, all, (size_t)c->nranks * bytes, s)) r = ncclSystemError;
    free(all);
    return r;
}
