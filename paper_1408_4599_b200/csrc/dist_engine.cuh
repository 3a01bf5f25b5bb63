// dist_engine.cuh -- spatial decomposition across GPUs (§4,
// P:189-252), included once by mardyn.cu (it uses the
// context's private helpers).
//
// A "group" is the set of ranks that step together: one per process, NCCL
// communicator owned by the library (mardyn_create_distributed), or all ranks
// inside one process on one device (mardyn_create_loopback: the correctness
// path on a single GPU, records moved by direct device stores).  Everything
// of the method happens here or in the kernels: the k-d partition from the
// Eq. 6 cell costs, the per-step halo exchange and
// migration, the rebalance from the measured per-cell
// loads every rebalance_interval steps, and the global
// observables as rank-ordered sums (reading A23).  The caller only launches
// ranks and steps them.

struct Group {
    int p = 1;
    bool nccl = false;
    ncclComm_t comm = nullptr;
    std::vector<mardyn_ctx*> m;          // loopback: every rank, in rank order; NCCL: this process's rank
    int live = 0;                        // contexts not yet destroyed
    cudaStream_t stream = nullptr;       // loopback: the one stream every rank enqueues on
    bool own_stream = false;
    std::vector<const ObsRec*> hist_tab; // loopback NVT: the ranks' observable rings (host staging)
    std::vector<std::pair<std::string, void*>> ipc_open;   // NCCL: peers' receive allocations opened (CUDA IPC)
    // the steady-state step of every local rank (begin halves, exchange, end halves) captured as
    // one CUDA graph per buffer parity; rebuilt when the segment layout, the partition, the
    // molecules or the profiling switch change
    cudaGraphExec_t gx[2] = {nullptr, nullptr};
};

static bool nccl_graphs()
{
    static const bool on = [] { const char* e = std::getenv("MARDYN_NCCL_GRAPHS"); return e && e[0] == '1'; }();
    return on;
}

static void group_drop_graphs(Group* G)
{
    if (!G) return;
    for (int b = 0; b < 2; ++b)
        if (G->gx[b]) { cudaGraphExecDestroy(G->gx[b]); G->gx[b] = nullptr; }
}

static bool group_is_nccl(const Group* g) { return g && g->nccl; }

// timing events of the decomposed step: recorded as external event nodes when the step is
// being captured into a graph (loopback, MARDYN_NCCL_GRAPHS=1), as plain records when it is
// enqueued eagerly (the NCCL step): cudaEventRecordExternal outside a capture is an error
static cudaError_t ev_record(cudaEvent_t e, cudaStream_t s)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const cudaError_t q = cudaStreamIsCapturing(s, &cs);
    if (q != cudaSuccess) return q;
    return cudaEventRecordWithFlags(e, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                             : cudaEventRecordDefault);
}
static std::vector<mardyn_ctx*> group_members(mardyn_ctx* ctx)
{
    std::vector<mardyn_ctx*> out;
    for (mardyn_ctx* c : ctx->grp ? ctx->grp->m : std::vector<mardyn_ctx*>{ctx})
        if (c) out.push_back(c);
    return out;
}

#define NCK(call)                                                                                    \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess) {                                                                     \
            ctx->poisoned = true;                                                                    \
            return fail(ctx, MARDYN_ENCCL, std::string(#call) + ": " + mdn::api().GetErrorString(r_)); \
        }                                                                                            \
    } while (0)

static void group_release(mardyn_ctx* ctx)
{
    Group* G = ctx->grp;
    if (!G) return;
    ctx->grp = nullptr;
    group_drop_graphs(G);                 // the graphs hold this rank's buffers
    for (auto& c : G->m)                  // the remaining ranks see a destroyed rank (group_ok)
        if (c == ctx) c = nullptr;
    if (--G->live > 0) return;
    for (auto& kv : G->ipc_open) cudaIpcCloseMemHandle(kv.second);
    if (G->comm) mdn::api().CommDestroy(G->comm);
    if (G->own_stream && G->stream) cudaStreamDestroy(G->stream);
    delete G;
}

// ---- host-side partition (every rank computes the same: deterministic host code)

// cell of a global position by the integer rules of reading A12 (as k_ingest)
static inline int64_t host_cell(const GridP& g, const double* r)
{
    int64_t c[3];
    for (int k = 0; k < 3; ++k) {
        const long long P = (long long)g.P64[k];
        long long x = llrint(r[k] / (double)g.s);
        x %= P;
        if (x < 0) x += P;
        c[k] = (int64_t)((uint64_t)x / g.E[k]);
    }
    return c[0] + (int64_t)g.nc[0] * (c[1] + (int64_t)g.nc[1] * c[2]);
}

// owner / halo maps and this rank's home box from p boxes (validated)
static int dd_set_maps(mardyn_ctx* ctx, const int32_t* boxes)
{
    const GridP& g0 = ctx->g;
    const int nx = g0.nc[0], ny = g0.nc[1], nz = g0.nc[2], p = ctx->nranks;
    std::vector<uint8_t> owner((size_t)g0.ncell, 255);
    for (int r = 0; r < p; ++r) {
        const int32_t* b = boxes + 6 * r;
        for (int k = 0; k < 3; ++k)
            if (b[k] < 0 || b[3 + k] > g0.nc[k] || b[3 + k] - b[k] < 2)
                return fail(ctx, MARDYN_EINVAL, "every box needs >= 2 cells per axis inside the grid (P:213)");
        for (int z = b[2]; z < b[5]; ++z)
            for (int y = b[1]; y < b[4]; ++y)
                for (int x = b[0]; x < b[3]; ++x) {
                    uint8_t& o = owner[x + (size_t)nx * (y + (size_t)ny * z)];
                    if (o != 255) return fail(ctx, MARDYN_EINVAL, "boxes overlap");
                    o = (uint8_t)r;
                }
    }
    for (uint8_t o : owner)
        if (o == 255) return fail(ctx, MARDYN_EINVAL, "boxes do not tile the grid");
    // halo of rank r: cells within one cell (periodic, edge >= rc) of its box owned by another rank
    std::vector<uint32_t> gmask((size_t)g0.ncell, 0u);
    for (int r = 0; r < p; ++r) {
        const int32_t* b = boxes + 6 * r;
        for (int z = b[2] - 1; z <= b[5]; ++z)
            for (int y = b[1] - 1; y <= b[4]; ++y)
                for (int x = b[0] - 1; x <= b[3]; ++x) {
                    const size_t c = (size_t)((x + nx) % nx) + (size_t)nx * (((y + ny) % ny) + (size_t)ny * ((z + nz) % nz));
                    if (owner[c] != r) gmask[c] |= 1u << r;
                }
    }
    ctx->boxes.assign(boxes, boxes + 6 * p);
    ctx->h_owner.swap(owner);
    ctx->h_gmask.swap(gmask);
    const int32_t* b = boxes + 6 * ctx->dd_rank;
    GridP& g = ctx->g;
    // the rank-local cell window: the box and one halo layer (the whole axis if that covers it)
    g.wncell = 1;
    for (int k = 0; k < 3; ++k) {
        g.hdim[k] = b[3 + k] - b[k];
        if (g.hdim[k] + 2 >= g.nc[k]) { g.wlo[k] = 0; g.wn[k] = g.nc[k]; }
        else { g.wlo[k] = (b[k] - 1 + g.nc[k]) % g.nc[k]; g.wn[k] = g.hdim[k] + 2; }
        g.hlo[k] = loc_axis(g, k, b[k]);
        g.wncell *= g.wn[k];
    }
    g.nhome = g.hdim[0] * g.hdim[1] * g.hdim[2];
    if (ctx->ws) {
        CK(cudaMemcpyAsync(ctx->owner, ctx->h_owner.data(), ctx->g.ncell, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->gmask, ctx->h_gmask.data(), 4 * (size_t)ctx->g.ncell, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return MARDYN_OK;
}

// k-d boxes from per-cell molecule counts: Eq. 6 cost (reading A19), recursive
// bisection with alternating axes and minimum-imbalance planes
static int boxes_from_counts(mardyn_ctx* ctx, const int32_t* counts, std::vector<int32_t>& boxes)
{
    const GridP& g = ctx->g;
    const int nx = g.nc[0], ny = g.nc[1], nz = g.nc[2], p = ctx->nranks;
    std::vector<double> cost((size_t)g.ncell);
    if (ctx->cost_model == 1)             // linear: the molecules per cell (mardyn_set_cost_model)
        for (size_t c = 0; c < cost.size(); ++c) cost[c] = (double)counts[c];
    else
        mdd::cell_cost(counts, nx, ny, nz, cost.data());
    std::vector<mdd::Box> leaves;
    mdd::Box all;
    all.lo[0] = all.lo[1] = all.lo[2] = 0;
    all.hi[0] = nx; all.hi[1] = ny; all.hi[2] = nz;
    if (!mdd::kd_split(cost.data(), nx, ny, all, p, 0, leaves) || (int)leaves.size() != p)
        return fail(ctx, MARDYN_EINVAL, "k-d decomposition: the 2-cell constraint cannot be met (P:213)");
    boxes.assign(6 * (size_t)p, 0);
    for (int r = 0; r < p; ++r)
        for (int k = 0; k < 3; ++k) { boxes[6 * r + k] = leaves[r].lo[k]; boxes[6 * r + 3 + k] = leaves[r].hi[k]; }
    return MARDYN_OK;
}

// ---- decomposed ingest (every rank reads the GLOBAL arrays, keeps owned + halo)

static int set_molecules_dd(mardyn_ctx* ctx, int64_t n, const int64_t* id, const int32_t* comp, const double* r,
                            const double* v, const double* q, const double* j, int32_t half_step)
{
    if (ctx->h_owner.empty()) return fail(ctx, MARDYN_ESTATE, "mardyn_partition (or set_partition) first");
    if (n < 1 || n > (1ll << 31) - 1) return fail(ctx, MARDYN_EINVAL, "n must be in [1, 2^31)");
    if (!comp || !r || !v) return fail(ctx, MARDYN_EINVAL, "comp, r, v are required");
    if (ctx->rigid && (!q || !j)) return fail(ctx, MARDYN_EINVAL, "q and j are required for rigid molecules");
    const int ncomp = (int)ctx->comps.size();
    ctx->ids.resize(n);
    ctx->comp_host.assign(comp, comp + n);
    for (int64_t i = 0; i < n; ++i) ctx->ids[i] = id ? id[i] : i;
    ctx->comp_counts.assign(ncomp, 0);
    double ndof = 3.0 * n;
    for (int64_t i = 0; i < n; ++i)
        if (comp[i] >= 0 && comp[i] < ncomp) {
            ctx->comp_counts[comp[i]] += 1;
            ndof += ctx->model.comp[comp[i]].rot;
        }
    ctx->ndof = ctx->ndof_global = ndof;      // T of the rank-local partials sums to the global T
    ctx->n_global = ctx->n_input = n;
    ctx->n_stale = false;
    group_drop_graphs(ctx->grp);
    ctx->seg_ready = false;
    ctx->peer_segs = false;
    ctx->direct = false;
    cudaStream_t s = ctx->stream;
    if (ctx->force_grid != ctx->force_blocks) {
        ctx->force_grid = ctx->force_blocks;
        CK(cudaMemsetAsync(ctx->fpart, 0, sizeof(ForcePartial) * ctx->nfpart, s));
    }
    CK(cudaMemsetAsync(ctx->count, 0, sizeof(int) * ctx->ncell_pad, s));
    CK(cudaMemsetAsync(ctx->flag, 0, 4, s));
    CK(cudaMemsetAsync(ctx->n_aux, 0, 16, s));
    // the global arrays in chunks through the staging area (r 24, v 24, q 32, j 24, comp 4 B)
    const int64_t chunk = std::min<int64_t>(n, ctx->cap);
    double* dr = (double*)ctx->stage;
    double* dv = dr + 3 * chunk;
    double* dq = dv + 3 * chunk;
    double* dj = dq + 4 * chunk;
    int* dc = (int*)(dj + 3 * chunk);
    const int src = 1, dst = 0;
    for (int64_t base = 0; base < n; base += chunk) {
        const int64_t m = std::min(chunk, n - base);
        CK(cudaMemcpyAsync(dr, r + 3 * base, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dv, v + 3 * base, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
        if (ctx->rigid) {
            CK(cudaMemcpyAsync(dq, q + 4 * base, sizeof(double) * 4 * m, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dj, j + 3 * base, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
        }
        CK(cudaMemcpyAsync(dc, comp + base, sizeof(int) * m, cudaMemcpyHostToDevice, s));
        k_ingest_dd<<<nblk(m, 256), 256, 0, s>>>((int)m, (int)base, dr, dv, ctx->rigid ? dq : nullptr,
                                                 ctx->rigid ? dj : nullptr, dc, ctx->g, ctx->pos[src], ctx->vel[src],
                                                 ctx->rigid ? ctx->quat[src] : nullptr,
                                                 ctx->rigid ? ctx->angm[src] : nullptr, ctx->cell_of, ctx->rank,
                                                 ctx->count, ncomp, ctx->flag, ctx->owner, ctx->gmask, ctx->dd_rank,
                                                 ctx->n_aux, (int)ctx->cap);
        ctx->launches += 1;
    }
    int hk[2] = {0, 0};
    CK(cudaMemcpyAsync(&hk[0], ctx->n_aux, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hk[1], ctx->flag, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hk[1] & (512 | 1024)) {
        ctx->loaded = false;
        CK(cudaMemsetAsync(ctx->flag, 0, 4, s));
        CK(cudaMemsetAsync(ctx->count, 0, sizeof(int) * ctx->ncell_pad, s));
        CK(cudaStreamSynchronize(s));
        if (hk[1] & 512)
            return fail(ctx, MARDYN_EINVAL, "invalid input: non-finite position or velocity, component id out of "
                                            "range, or non-unit quaternion");
        return fail(ctx, MARDYN_ECAPACITY, "owned + halo molecules of this rank exceed the capacity (" +
                                               std::to_string(hk[0]) + " > " + std::to_string(ctx->cap) + ")");
    }
    ctx->n = hk[0];
    int rc = enqueue_sort(ctx, src, dst, ctx->n);
    if (rc) return rc;
    ctx->cur = dst;
    long long step = ctx->host_step;
    CK(cudaMemcpyAsync(ctx->step_ctr, &step, 8, cudaMemcpyHostToDevice, s));
    if (!half_step) {   // A8: backward half kick with F(t0), tau(t0) (halo copies are kicked by their owners)
        launch_force(ctx, ctx->cur);
        const int nk = (int)ctx->n;
        if (ctx->rigid)
            k_half_kick<true><<<nblk(nk, 256), 256, 0, s>>>(nk, ctx->g, ctx->dmodel, ctx->vel[ctx->cur],
                                                            ctx->angm[ctx->cur], ctx->force, ctx->torque);
        else
            k_half_kick<false><<<nblk(nk, 256), 256, 0, s>>>(nk, ctx->g, ctx->dmodel, ctx->vel[ctx->cur], nullptr,
                                                             ctx->force, nullptr);
        ctx->launches += 1;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    ctx->loaded = true;
    ctx->last_obs = -1;
    return MARDYN_OK;
}

// owned molecules of this rank, compacted on the device, ordered by global index on the host
static int egress_dd(mardyn_ctx* ctx, double* r, double* v, double* q, double* j, double* F, double* tau,
                     uint32_t* ufix, int32_t* cell, int64_t n_slots, int64_t* n_out, int64_t* ids_out,
                     int32_t* comp_out)
{
    const int64_t n = n_slots < 0 ? ctx->n : n_slots;
    cudaStream_t s = ctx->stream;
    const unsigned fields = (r ? 1u : 0u) | (v ? 2u : 0u) | (q ? 4u : 0u) | (j ? 8u : 0u) | (F ? 16u : 0u) |
                            (tau ? 32u : 0u) | (ufix ? 64u : 0u) | (cell ? 128u : 0u);
    const int widths[8] = {3, 3, 4, 3, 3, 3, 3, 1};
    int rw = 1;
    for (int k = 0; k < 8; ++k) if (fields >> k & 1u) rw += widths[k];
    double* out = (double*)ctx->stage;
    CK(cudaMemsetAsync(ctx->n_aux + 2, 0, 4, s));
    const int b = ctx->cur;
    k_egress_dd<<<nblk(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(
        (int)n, ctx->g, ctx->pos[b], ctx->vel[b], ctx->rigid ? ctx->quat[b] : nullptr,
        ctx->rigid ? ctx->angm[b] : nullptr, ctx->force, ctx->rigid ? ctx->torque : nullptr, fields, rw, out,
        ctx->n_aux + 2);
    ctx->launches += 1;
    int m = 0;
    CK(cudaMemcpyAsync(&m, ctx->n_aux + 2, 4, cudaMemcpyDeviceToHost, s));
    int rc = sync_check(ctx);
    if (rc) return rc;
    std::vector<double> h((size_t)m * rw);
    CK(cudaMemcpy(h.data(), out, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
    std::vector<int64_t> order(m);
    for (int k = 0; k < m; ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t c) { return h[a * rw] < h[c * rw]; });
    for (int t = 0; t < m; ++t) {
        const double* x = h.data() + order[t] * rw;
        const int64_t iid = (int64_t)x[0];
        int w = 1;
        if (r) { for (int k = 0; k < 3; ++k) r[3 * t + k] = x[w + k]; w += 3; }
        if (v) { for (int k = 0; k < 3; ++k) v[3 * t + k] = x[w + k]; w += 3; }
        if (q) { for (int k = 0; k < 4; ++k) q[4 * t + k] = x[w + k]; w += 4; }
        if (j) { for (int k = 0; k < 3; ++k) j[3 * t + k] = x[w + k]; w += 3; }
        if (F) { for (int k = 0; k < 3; ++k) F[3 * t + k] = x[w + k]; w += 3; }
        if (tau) { for (int k = 0; k < 3; ++k) tau[3 * t + k] = x[w + k]; w += 3; }
        if (ufix) { for (int k = 0; k < 3; ++k) ufix[3 * t + k] = (uint32_t)x[w + k]; w += 3; }
        if (cell) { cell[t] = (int32_t)x[w]; w += 1; }
        if (ids_out) ids_out[t] = ctx->ids[iid];
        if (comp_out) comp_out[t] = ctx->comp_host[iid];
    }
    if (n_out) *n_out = m;
    return MARDYN_OK;
}

// ---- one rank's halves of a step

static DDArgs dd_args(mardyn_ctx* ctx, bool uniform_max)
{
    DDArgs dd;
    dd.rank = ctx->dd_rank; dd.nranks = ctx->nranks; dd.owner = ctx->owner; dd.gmask = ctx->gmask;
    dd.send = ctx->sendbuf; dd.send_cnt = ctx->send_cnt; dd.flag = ctx->flag;
    dd.n_dev = nullptr;
    if (uniform_max) {                      // synchronous steps: uniform segments of the layout's stride
        dd.seg_cap = (int)ctx->seg_max;
        dd.seg_tab = nullptr;
    } else {
        dd.seg_cap = (int)ctx->seg_cap;
        dd.seg_tab = ctx->peer_segs ? ctx->seg_tab : nullptr;
    }
    dd.put_rec = nullptr;
    return dd;
}

// forces at t_k on the home box, kick / drift / rotation of the owned molecules, binning,
// records for the exchange (uniform segments, counts to the host)
static int dd_begin_sync(mardyn_ctx* ctx, int64_t* send_counts)
{
    if (int rc0 = refresh_n(ctx)) return rc0;
    cudaStream_t s = ctx->stream;
    const int b = ctx->cur, n = (int)ctx->n;
    long long step = ctx->host_step;
    CK(cudaMemcpyAsync(ctx->step_ctr, &step, 8, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(ctx->ev_f0[b], s));
    launch_force(ctx, b);
    CK(cudaEventRecord(ctx->ev_f1[b], s));
    CK(cudaMemsetAsync(ctx->count, 0, sizeof(int) * ctx->ncell_pad, s));
    CK(cudaMemsetAsync(ctx->send_cnt, 0, sizeof(int) * ctx->nranks, s));
    DDArgs dd = dd_args(ctx, true);
    const int nkb = nblk(std::max(n, 1), 256);
    if (ctx->rigid)
        k_integrate<true, true><<<nkb, 256, 0, s>>>(n, ctx->g, ctx->dmodel, ctx->pos[b], ctx->vel[b], ctx->quat[b],
                                                    ctx->angm[b], ctx->force, ctx->torque, ctx->cell_of, ctx->rank,
                                                    ctx->count, ctx->kpart, ctx->flag, dd);
    else
        k_integrate<false, true><<<nkb, 256, 0, s>>>(n, ctx->g, ctx->dmodel, ctx->pos[b], ctx->vel[b], nullptr,
                                                     nullptr, ctx->force, ctx->torque, ctx->cell_of, ctx->rank,
                                                     ctx->count, ctx->kpart, ctx->flag, dd);
    k_finalize<<<FIN_BLOCKS, FIN_THREADS, 0, s>>>(ctx->nfpart, ctx->fpart, nkb, ctx->kpart, ctx->ndof,
                                                  ctx->step_ctr, 1, ctx->hist, ctx->fin_scratch, ctx->fin_ticket, 0);
    ctx->launches += 3;
    CK(cudaGetLastError());
    std::vector<int> cnt(ctx->nranks);
    CK(cudaMemcpyAsync(cnt.data(), ctx->send_cnt, 4 * ctx->nranks, cudaMemcpyDeviceToHost, s));
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, ctx->flag, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (flag & 256) return fail(ctx, MARDYN_ECAPACITY, "exchange segment overflow");
    for (int r = 0; r < ctx->nranks; ++r) send_counts[r] = cnt[r];
    ctx->last_parity = b;
    return MARDYN_OK;
}

// import the n_recv records at the start of the receive buffer, rebuild the cells
static int dd_import_sort(mardyn_ctx* ctx, int64_t n_recv, bool advance)
{
    if (n_recv < 0 || n_recv > ctx->recv_cap || ctx->n + n_recv > ctx->cap)
        return fail(ctx, MARDYN_ECAPACITY, "received records exceed the capacity");
    cudaStream_t s = ctx->stream;
    const int b = ctx->cur;
    if (n_recv > 0) {
        k_import<<<nblk(n_recv, 256), 256, 0, s>>>((int)n_recv, (int)ctx->n, ctx->g, ctx->recvbuf, ctx->pos[b],
                                                   ctx->vel[b], ctx->rigid ? ctx->quat[b] : nullptr,
                                                   ctx->rigid ? ctx->angm[b] : nullptr, ctx->cell_of, ctx->rank,
                                                   ctx->count);
        ctx->launches += 1;
    }
    int rc = enqueue_sort(ctx, b, 1 - b, ctx->n + n_recv);
    if (rc) return rc;
    CK(cudaGetLastError());
    int kept = 0;
    CK(cudaMemcpyAsync(&kept, ctx->start + ctx->g.wncell, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->n = kept;
    ctx->cur = 1 - b;
    if (advance) {
        ctx->host_step += 1;
        ctx->last_obs = ctx->host_step - 1;
    }
    return MARDYN_OK;
}

// asynchronous step (no host synchronisation): records packed into fixed per-peer
// segments (or stored straight into the receiving rank's buffer: direct puts), counts in
// device memory
static int dd_begin_async(mardyn_ctx* ctx)
{
    cudaStream_t s = ctx->stream;
    const int b = ctx->cur;
    DDArgs dd = dd_args(ctx, false);
    dd.n_dev = ctx->start + ctx->g.wncell;             // the sorted count of the last cell rebuild
    dd.put_rec = ctx->direct ? ctx->put_rec : nullptr;
    dd.peer_puts = ctx->direct && ctx->grp && ctx->grp->nccl;    // IPC puts into other processes / GPUs
    // (send_cnt is zero here: the last import cleared it)
    if (ctx->kernel == KER_LJ1) {
        // single-site kernel with the leapfrog, binning and exchange packing fused in (the cell
        // counts are zero: the last rebuild's scan cleared them); it also records its sorted
        // count and, with direct puts, stores the record counts into the receivers
        dd.n_force = ctx->n_aux + 1;
        dd.put_cnt = ctx->direct ? ctx->put_cnt : nullptr;
        dd.done = ctx->n_aux + 3;
        CK(ev_record(ctx->ev_f0[b], s));
        launch_force(ctx, b, true, true, &dd);
        CK(ev_record(ctx->ev_f1[b], s));
        // the step's observables on a side stream, concurrent with the exchange and the rebuild
        CK(cudaEventRecord(ctx->ev_s0, s));
        CK(cudaStreamWaitEvent(ctx->side_stream, ctx->ev_s0, 0));
        k_finalize<<<FIN_BLOCKS, FIN_THREADS, 0, ctx->side_stream>>>(ctx->nfpart, ctx->fpart, 0, ctx->kpart,
                                                                     ctx->ndof, ctx->step_ctr, 1, ctx->hist,
                                                                     ctx->fin_scratch, ctx->fin_ticket, 0);
        CK(cudaEventRecord(ctx->ev_s1, ctx->side_stream));
        ctx->side_join = true;
        ctx->launches += 1;
        CK(cudaGetLastError());
        ctx->last_parity = b;
        return MARDYN_OK;
    }
    CK(cudaMemcpyAsync(ctx->n_aux + 1, ctx->start + ctx->g.wncell, 4, cudaMemcpyDeviceToDevice, s));
    CK(ev_record(ctx->ev_f0[b], s));
    launch_force(ctx, b, false, true);
    CK(ev_record(ctx->ev_f1[b], s));
    CK(cudaMemsetAsync(ctx->count, 0, sizeof(int) * ctx->ncell_pad, s));
    const int nkb = ctx->nkblocks;
    if (ctx->rigid)
        k_integrate<true, true><<<nkb, 256, 0, s>>>((int)ctx->cap, ctx->g, ctx->dmodel, ctx->pos[b], ctx->vel[b],
                                                    ctx->quat[b], ctx->angm[b], ctx->force, ctx->torque, ctx->cell_of,
                                                    ctx->rank, ctx->count, ctx->kpart, ctx->flag, dd);
    else
        k_integrate<false, true><<<nkb, 256, 0, s>>>((int)ctx->cap, ctx->g, ctx->dmodel, ctx->pos[b], ctx->vel[b],
                                                     nullptr, nullptr, ctx->force, ctx->torque, ctx->cell_of,
                                                     ctx->rank, ctx->count, ctx->kpart, ctx->flag, dd);
    if (ctx->direct) {
        k_put_counts<<<1, 32, 0, s>>>(ctx->nranks, ctx->send_cnt, ctx->put_cnt);
        ctx->launches += 1;
    }
    k_finalize<<<FIN_BLOCKS, FIN_THREADS, 0, s>>>(ctx->nfpart, ctx->fpart, nkb, ctx->kpart, ctx->ndof,
                                                  ctx->step_ctr, 1, ctx->hist, ctx->fin_scratch, ctx->fin_ticket, 0);
    ctx->launches += 3;
    CK(cudaGetLastError());
    ctx->last_parity = b;
    return MARDYN_OK;
}

static int dd_end_async(mardyn_ctx* ctx)
{
    cudaStream_t s = ctx->stream;
    const int b = ctx->cur;
    const int seg = (int)ctx->seg_cap;
    const int64_t span = ctx->peer_segs ? ctx->recv_span : (int64_t)seg * ctx->nranks;
    k_import_seg<<<nblk(span, 256), 256, 0, s>>>(
        ctx->nranks, seg, ctx->peer_segs ? ctx->seg_tab + 2 * ctx->nranks : nullptr, ctx->recv_cnt,
        ctx->start + ctx->g.wncell, (int)ctx->cap, ctx->g, ctx->recvbuf, ctx->pos[b], ctx->vel[b],
        ctx->rigid ? ctx->quat[b] : nullptr, ctx->rigid ? ctx->angm[b] : nullptr, ctx->cell_of, ctx->rank,
        ctx->count, ctx->n_aux, ctx->flag, ctx->send_cnt);
    ctx->launches += 1;
    int rc = enqueue_sort(ctx, b, 1 - b, -1, ctx->n_aux);
    if (rc) return rc;
    if (ctx->side_join) {                              // the next step's force rewrites the partials
        CK(cudaStreamWaitEvent(s, ctx->ev_s1, 0));
        ctx->side_join = false;
    }
    CK(cudaGetLastError());
    ctx->n_stale = true;
    ctx->cur = 1 - b;
    ctx->host_step += 1;
    ctx->last_obs = ctx->host_step - 1;
    return MARDYN_OK;
}

// per-peer segment layout (device table + host copies)
static int dd_set_segments(mardyn_ctx* ctx, const std::vector<int64_t>& sc, const std::vector<int64_t>& rcap)
{
    const int p = ctx->nranks;
    std::vector<int> tab(4 * (size_t)p);
    ctx->send_off.assign(p, 0); ctx->recv_off.assign(p, 0);
    int64_t so = 0, ro = 0;
    for (int r = 0; r < p; ++r) {
        tab[r] = (int)so; tab[p + r] = (int)sc[r];
        tab[2 * p + r] = (int)ro; tab[3 * p + r] = (int)rcap[r];
        ctx->send_off[r] = so; ctx->recv_off[r] = ro;
        so += sc[r];
        ro += rcap[r];
    }
    ctx->send_caps = sc;
    ctx->recv_caps = rcap;
    CK(cudaMemcpyAsync(ctx->seg_tab, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->recv_cnt, 0, sizeof(int) * p, ctx->stream));
    CK(cudaMemsetAsync(ctx->send_cnt, 0, sizeof(int) * p, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->peer_segs = true;
    ctx->seg_cap = 0;
    ctx->recv_span = ro;
    return MARDYN_OK;
}

// ---- the group's steps

// A rank that fails before a collective and returns would leave its peers waiting in that
// collective.  Before each collective of the host-synchronous paths (first step, rebalance,
// observables) the ranks therefore agree on the outcome: a one-word ncclAllReduce(max) of
// "this rank failed"; every rank then returns an error.  (A poisoned context cannot enqueue
// anything; its peers stop at their next NCCL call.)
static int group_agree(Group* G, int rc)
{
    if (!G || !G->nccl || G->p < 2) return rc;
    mardyn_ctx* ctx = G->m[0];
    if (ctx->poisoned || !ctx->cmat) return rc;
    int32_t* d = reinterpret_cast<int32_t*>(ctx->cmat + (size_t)G->p * (G->p + 1));
    int32_t h = rc != MARDYN_OK ? 1 : 0;
    CK(cudaMemcpyAsync(d, &h, 4, cudaMemcpyHostToDevice, ctx->stream));
    NCK(mdn::api().AllReduce(d, d, 1, ncclInt32, ncclMax, G->comm, ctx->stream));
    CK(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (rc != MARDYN_OK) return rc;
    if (h) return fail(ctx, MARDYN_ESTATE, "another rank of the decomposition failed");
    return MARDYN_OK;
}

// the record-count matrix C[src][dst] of every rank (allgather over NCCL, or read across the
// loopback ranks); rows = this process's ranks' counts
static int gather_counts(Group* G, std::vector<std::vector<int64_t>>& C)
{
    const int p = G->p;
    if (!G->nccl) return MARDYN_OK;                    // loopback: every row is local already
    mardyn_ctx* ctx = G->m[0];
    const int me = ctx->dd_rank;
    int64_t* row = ctx->cmat + (size_t)p * p;
    CK(cudaMemcpyAsync(row, C[me].data(), 8 * (size_t)p, cudaMemcpyHostToDevice, ctx->stream));
    NCK(mdn::api().AllGather(row, ctx->cmat, (size_t)p, ncclInt64, G->comm, ctx->stream));
    std::vector<int64_t> all((size_t)p * p);
    CK(cudaMemcpyAsync(all.data(), ctx->cmat, 8 * all.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < p; ++r)
        for (int d = 0; d < p; ++d) C[r][d] = all[(size_t)r * p + d];
    return MARDYN_OK;
}

// move the counted records (src's segment dst at send_off[dst] -> dst's receive buffer,
// contiguous in source order); returns per local rank the records received
static int exchange_exact(Group* G, const std::vector<std::vector<int64_t>>& C, std::vector<int64_t>& nrecv)
{
    NvtxRange nvtx_range("dd_exchange");
    const int p = G->p;
    const size_t RB = sizeof(DDRec);
    nrecv.assign(p, 0);
    if (!G->nccl) {
        for (mardyn_ctx* dst : G->m) {
            mardyn_ctx* ctx = dst;
            const int d = dst->dd_rank;
            int64_t off = 0;
            for (mardyn_ctx* src : G->m) {
                const int64_t k = C[src->dd_rank][d];
                if (k) CK(cudaMemcpyAsync(dst->recvbuf + off, src->sendbuf + src->send_off[d], k * RB,
                                          cudaMemcpyDeviceToDevice, dst->stream));
                off += k;
            }
            nrecv[d] = off;
        }
        return MARDYN_OK;
    }
    mardyn_ctx* ctx = G->m[0];
    const int me = ctx->dd_rank;
    int64_t off = 0;
    std::vector<int64_t> roff(p);
    for (int r = 0; r < p; ++r) { roff[r] = off; off += C[r][me]; }
    nrecv[me] = off;
    if (C[me][me]) return fail(ctx, MARDYN_ESTATE, "records addressed to the sending rank");
    NCK(mdn::api().GroupStart());
    for (int d = 0; d < p; ++d) {
        if (d == me) continue;
        if (C[me][d]) NCK(mdn::api().Send(ctx->sendbuf + ctx->send_off[d], C[me][d] * RB, ncclChar, d, G->comm, ctx->stream));
        if (C[d][me]) NCK(mdn::api().Recv(ctx->recvbuf + roff[d], C[d][me] * RB, ncclChar, d, G->comm, ctx->stream));
    }
    NCK(mdn::api().GroupEnd());
    return MARDYN_OK;
}

// NCCL groups: this step's receive area, count array and put tables (parity = cur: every rank
// flips cur once per step, so the ranks agree on it)
static void nccl_parity(Group* G)
{
    if (!G || !G->nccl || G->p < 2) return;
    for (mardyn_ctx* c : G->m) {
        const int b = c->cur & 1;
        c->recvbuf = c->recv_area[b];
        c->recv_cnt = c->rcnt_area[b];
        c->put_rec = c->put_rec_area[b];
        c->put_cnt = c->put_cnt_area[b];
    }
}

static bool ipc_puts_enabled()
{
    static const bool on = [] { const char* e = std::getenv("MARDYN_IPC_PUTS"); return !(e && e[0] == '0'); }();
    return on;
}

// Direct puts across processes (GPUs): every rank exports the allocation holding its two
// receive areas as a CUDA IPC handle, the handles, offsets and receive-segment layouts are
// all-gathered over the communicator, and every rank opens its peers' allocations (over
// NVLink peer mappings on a multi-GPU node).  The packing kernels then store each record
// straight into its receiver's area of this step's parity, and the count of records into the
// receiver's count array, while the force + leapfrog kernel produces them -- the transfer
// overlaps the computation -- and one stream-ordered one-word all-reduce per step orders
// every rank's stores before every rank's import.  Two areas per rank: a peer that has
// passed step k's all-reduce stores step k + 1's records into the other area while this rank
// still imports step k's.  Taken only when every rank could export and open (agreed by an
// all-reduce); otherwise, or with MARDYN_IPC_PUTS=0, the records move by grouped send / recv.
static int nccl_ipc_setup(Group* G)
{
    mardyn_ctx* ctx = G->m[0];
    const int p = G->p, me = ctx->dd_rank;
    ctx->direct = false;
    if (!G->nccl || p < 2 || !ipc_puts_enabled() || !ctx->ipc_blob || !ctx->ipc_word) return MARDYN_OK;
    cudaStream_t s = ctx->stream;
    const size_t B = ipc_blob_bytes(p);
    std::vector<char> mine(B, 0), all(B * (size_t)p);
    typedef int (*AddrRange)(unsigned long long*, size_t*, unsigned long long);
    static const AddrRange range = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return reinterpret_cast<AddrRange>(f);
    }();
    unsigned long long base = 0;
    size_t asize = 0;
    int64_t ok = 0;
    cudaIpcMemHandle_t h;
    if (range && range(&base, &asize, (unsigned long long)(uintptr_t)ctx->recv_area[0]) == 0 &&
        cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base) == cudaSuccess) {
        ok = 1;
        std::memcpy(mine.data(), &h, 64);
    } else {
        cudaGetLastError();
    }
    int64_t* w = reinterpret_cast<int64_t*>(mine.data() + 64);
    w[0] = ok;
    w[1] = (int64_t)((uintptr_t)ctx->recv_area[0] - base);
    w[2] = (int64_t)((uintptr_t)ctx->recv_area[1] - base);
    w[3] = (int64_t)((uintptr_t)ctx->rcnt_area[0] - base);
    w[4] = (int64_t)((uintptr_t)ctx->rcnt_area[1] - base);
    for (int r = 0; r < p; ++r) w[5 + r] = ctx->recv_off[r];
    char* slot = ctx->ipc_blob + (size_t)me * B;
    CK(cudaMemcpyAsync(slot, mine.data(), B, cudaMemcpyHostToDevice, s));
    NCK(mdn::api().AllGather(slot, ctx->ipc_blob, B, ncclChar, G->comm, s));
    CK(cudaMemcpyAsync(all.data(), ctx->ipc_blob, B * (size_t)p, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<uint64_t> tab(4 * (size_t)p);          // [q][dst] record base, [q][dst] count word
    int32_t good = 1;
    for (int d = 0; d < p && good; ++d) {
        const char* e = all.data() + (size_t)d * B;
        const int64_t* v = reinterpret_cast<const int64_t*>(e + 64);
        if (!v[0]) { good = 0; break; }
        char* pb = nullptr;
        if (d == me) {
            pb = (char*)(uintptr_t)base;
        } else {
            const std::string key(e, 64);
            for (auto& kv : G->ipc_open)
                if (kv.first == key) pb = (char*)kv.second;
            if (!pb) {
                cudaIpcMemHandle_t hd;
                std::memcpy(&hd, e, 64);
                void* ptr = nullptr;
                if (cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    good = 0;
                    break;
                }
                G->ipc_open.emplace_back(key, ptr);
                pb = (char*)ptr;
            }
        }
        for (int q = 0; q < 2; ++q) {
            tab[(size_t)q * 2 * p + d] = (uint64_t)(uintptr_t)(pb + v[1 + q]) + sizeof(DDRec) * (uint64_t)v[5 + me];
            tab[(size_t)q * 2 * p + p + d] = (uint64_t)(uintptr_t)(pb + v[3 + q]) + 4 * (uint64_t)me;
        }
    }
    // every rank takes the direct path, or none does
    CK(cudaMemcpyAsync(ctx->ipc_word, &good, 4, cudaMemcpyHostToDevice, s));
    NCK(mdn::api().AllReduce(ctx->ipc_word, ctx->ipc_word, 1, ncclInt32, ncclMin, G->comm, s));
    CK(cudaMemcpyAsync(&good, ctx->ipc_word, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!good) return MARDYN_OK;
    for (int q = 0; q < 2; ++q) {
        CK(cudaMemcpyAsync(ctx->put_rec_area[q], tab.data() + (size_t)q * 2 * p, 8 * (size_t)p,
                           cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->put_cnt_area[q], tab.data() + (size_t)q * 2 * p + p, 8 * (size_t)p,
                           cudaMemcpyHostToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
    ctx->direct = true;
    return MARDYN_OK;
}

// first step after a load or a rebalance: record counts to the host, exact exchange, then the
// per-peer segments of the asynchronous steps (twice the count + 1024 records: face
// neighbours send far more than edge or corner ones); loopback ranks get direct puts
static int group_sync_step(Group* G)
{
    NvtxRange nvtx_range("dd_sync_step");
    const int p = G->p;
    group_drop_graphs(G);                 // the segment layout is about to change
    nccl_parity(G);
    for (mardyn_ctx* c : G->m) c->rank_timed = false;
    std::vector<std::vector<int64_t>> C(p, std::vector<int64_t>(p, 0));
    for (mardyn_ctx* c : G->m) {
        if (int rc = group_agree(G, dd_begin_sync(c, C[c->dd_rank].data()))) return rc;
        c->send_off.assign(p, 0);
        for (int d = 0; d < p; ++d) c->send_off[d] = (int64_t)d * c->seg_max;   // uniform segments
    }
    if (int rc = gather_counts(G, C)) return rc;
    std::vector<int64_t> nrecv;
    if (int rc = exchange_exact(G, C, nrecv)) return rc;
    for (mardyn_ctx* c : G->m)
        if (int rc = group_agree(G, dd_import_sort(c, nrecv[c->dd_rank], true))) return rc;
    // segment capacities from the global count matrix (the same decision on every rank)
    auto capof = [](int64_t c) { return ((2 * c + 1024 + 255) / 256) * 256; };
    bool fits = true;
    mardyn_ctx* c0 = G->m[0];
    for (int r = 0; r < p; ++r) {
        int64_t ss = 0, rs = 0;
        for (int d = 0; d < p; ++d) { ss += capof(C[r][d]); rs += capof(C[d][r]); }
        fits = fits && ss <= c0->seg_max * p && rs <= c0->recv_cap;
    }
    int64_t big = 0;
    for (int r = 0; r < p; ++r)
        for (int d = 0; d < p; ++d) big = std::max(big, capof(C[r][d]));
    const int64_t useg = std::min({c0->seg_max, c0->recv_cap / p, big});
    for (mardyn_ctx* c : G->m) {
        const int r = c->dd_rank;
        std::vector<int64_t> sc(p), rc(p);
        for (int d = 0; d < p; ++d) {
            sc[d] = fits ? capof(C[r][d]) : useg;
            rc[d] = fits ? capof(C[d][r]) : useg;
            if (d == r) sc[d] = rc[d] = fits ? 256 : useg;
        }
        if (int e = dd_set_segments(c, sc, rc)) return e;
        c->seg_ready = true;
        c->direct = false;
    }
    if (!G->nccl) {                 // direct puts between the loopback ranks (one stream orders them)
        for (mardyn_ctx* src : G->m) {
            mardyn_ctx* ctx = src;
            std::vector<uint64_t> tab(2 * (size_t)p);
            for (mardyn_ctx* dst : G->m) {
                tab[dst->dd_rank] = (uint64_t)(uintptr_t)(dst->recvbuf + dst->recv_off[src->dd_rank]);
                tab[p + dst->dd_rank] = (uint64_t)(uintptr_t)(dst->recv_cnt + src->dd_rank);
            }
            CK(cudaMemcpyAsync(src->put_rec, tab.data(), sizeof(uint64_t) * p, cudaMemcpyHostToDevice, src->stream));
            CK(cudaMemcpyAsync(src->put_cnt, tab.data() + p, sizeof(uint64_t) * p, cudaMemcpyHostToDevice,
                               src->stream));
            CK(cudaStreamSynchronize(src->stream));
            src->direct = true;
        }
    } else if (int rc = nccl_ipc_setup(G)) {
        return rc;
    }
    return MARDYN_OK;
}

// steady-state step: no host synchronisation.  NCCL: the fixed segments and their counts as
// grouped send / recv on the context stream; loopback: the packing kernels already stored them.
// Enqueued once per buffer parity under stream capture and replayed as a CUDA graph.
static int group_async_enqueue(Group* G)
{
    nccl_parity(G);
    for (mardyn_ctx* c : G->m) {
        mardyn_ctx* ctx = c;
        if (c->profiling) CK(ev_record(c->ev_r[0], c->stream));
        if (int rc = dd_begin_async(c)) return rc;
        if (c->profiling) CK(ev_record(c->ev_r[1], c->stream));
    }
    if (G->nccl) {
        mardyn_ctx* ctx = G->m[0];
        const int p = G->p, me = ctx->dd_rank;
        const size_t RB = sizeof(DDRec);
        if (ctx->direct) {
            // records and counts are already in the receivers' areas (IPC puts): this one-word
            // all-reduce, stream-ordered after every rank's packing kernels, orders them
            // before every rank's import
            NCK(mdn::api().AllReduce(ctx->ipc_word, ctx->ipc_word, 1, ncclInt32, ncclSum, G->comm, ctx->stream));
        } else {
        NCK(mdn::api().GroupStart());
        for (int d = 0; d < p; ++d) {
            if (d == me) continue;
            NCK(mdn::api().Send(ctx->sendbuf + ctx->send_off[d], ctx->send_caps[d] * RB, ncclChar, d, G->comm, ctx->stream));
            NCK(mdn::api().Recv(ctx->recvbuf + ctx->recv_off[d], ctx->recv_caps[d] * RB, ncclChar, d, G->comm, ctx->stream));
            NCK(mdn::api().Send(ctx->send_cnt + d, 1, ncclInt32, d, G->comm, ctx->stream));
            NCK(mdn::api().Recv(ctx->recv_cnt + d, 1, ncclInt32, d, G->comm, ctx->stream));
        }
        NCK(mdn::api().GroupEnd());
        }
    }
    for (mardyn_ctx* c : G->m) {
        mardyn_ctx* ctx = c;
        if (c->profiling) CK(ev_record(c->ev_r[2], c->stream));
        if (int rc = dd_end_async(c)) return rc;
        if (c->profiling) CK(ev_record(c->ev_r[3], c->stream));
        c->rank_timed = c->profiling;
    }
    return MARDYN_OK;
}

static int group_async_step(Group* G)
{
    NvtxRange nvtx_range("dd_async_step");
    mardyn_ctx* ctx = G->m[0];
    cudaStream_t s = ctx->stream;             // loopback: every rank's stream; NCCL: the one rank's
    const int b = ctx->cur;
    // NCCL p2p under stream capture has not run on several GPUs here (one GPU this round): the
    // NCCL step stays eager unless MARDYN_NCCL_GRAPHS=1
    if (G->nccl && !nccl_graphs()) return group_async_enqueue(G);
    if (G->gx[b]) {
        CK(cudaGraphLaunch(G->gx[b], s));
        for (mardyn_ctx* c : G->m) {           // the host-side bookkeeping of begin / end
            c->last_parity = c->cur;
            c->cur = 1 - c->cur;
            c->n_stale = true;
            c->side_join = false;
            c->host_step += 1;
            c->last_obs = c->host_step - 1;
            c->rank_timed = c->profiling;
        }
        for (mardyn_ctx* c : G->m) c->launches += c->dd_glaunch;
        return MARDYN_OK;
    }
    // capture this parity's step (the capture pass performs the host bookkeeping itself)
    std::vector<long long> l0;
    for (mardyn_ctx* c : G->m) l0.push_back(c->launches);
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int rc = group_async_enqueue(G);
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (rc) return rc;
    CK(e);
    cudaGraphExec_t gx = nullptr;
    CK(cudaGraphInstantiate(&gx, graph, 0));
    CK(cudaGraphDestroy(graph));
    G->gx[b] = gx;
    for (size_t r = 0; r < G->m.size(); ++r) G->m[r]->dd_glaunch = G->m[r]->launches - l0[r];
    CK(cudaGraphLaunch(gx, s));
    return MARDYN_OK;
}

// Rebalance: measured per-cell loads of the last rebuild -> (allreduce) global
// counts -> Eq. 6 + k-d tree on the host (identical on every rank) -> new maps -> every
// rank re-distributes its owned molecules through exchange records
static int group_rebalance(Group* G)
{
    NvtxRange nvtx_range("dd_rebalance");
    const int p = G->p;
    group_drop_graphs(G);
    nccl_parity(G);
    mardyn_ctx* c0 = G->m[0];
    const int ncell = c0->g.ncell;
    std::vector<int32_t> counts((size_t)ncell, 0), tmp((size_t)ncell);
    for (mardyn_ctx* c : G->m) {
        mardyn_ctx* ctx = c;
        if (int rc = group_agree(G, refresh_n(c))) return rc;
        CK(cudaMemsetAsync(c->gcount, 0, 4 * (size_t)ncell, c->stream));
        k_owned_counts<<<nblk(c->g.wncell, 256), 256, 0, c->stream>>>(c->g, c->start, c->owner, c->dd_rank, c->gcount);
        c->launches += 1;
        CK(cudaGetLastError());
    }
    if (G->nccl) {
        mardyn_ctx* ctx = c0;
        NCK(mdn::api().AllReduce(c0->gcount, c0->gcount, (size_t)ncell, ncclInt32, ncclSum, G->comm, c0->stream));
        CK(cudaMemcpyAsync(counts.data(), c0->gcount, 4 * (size_t)ncell, cudaMemcpyDeviceToHost, c0->stream));
        CK(cudaStreamSynchronize(c0->stream));
    } else {
        for (mardyn_ctx* c : G->m) {
            mardyn_ctx* ctx = c;
            CK(cudaMemcpyAsync(tmp.data(), c->gcount, 4 * (size_t)ncell, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            for (int k = 0; k < ncell; ++k) counts[k] += tmp[k];
        }
    }
    std::vector<int32_t> boxes;
    if (int rc = boxes_from_counts(c0, counts.data(), boxes)) return rc;
    for (mardyn_ctx* c : G->m)
        if (int rc = dd_set_maps(c, boxes.data())) return rc;
    // redistribution: count the records per destination, lay them out exactly, pack, exchange
    std::vector<std::vector<int64_t>> C(p, std::vector<int64_t>(p, 0));
    for (mardyn_ctx* c : G->m) {
        mardyn_ctx* ctx = c;
        cudaStream_t s = c->stream;
        const int n = (int)c->n, b = c->cur;
        CK(cudaMemsetAsync(c->send_cnt, 0, sizeof(int) * p, s));
        DDArgs dd = dd_args(c, true);
        k_repartition<true><<<nblk(std::max(n, 1), 256), 256, 0, s>>>(n, c->g, dd, c->pos[b], c->vel[b],
                                                                       c->rigid ? c->quat[b] : nullptr,
                                                                       c->rigid ? c->angm[b] : nullptr,
                                                                       c->cell_of, c->rank, c->count);
        std::vector<int> cnt(p);
        CK(cudaMemcpyAsync(cnt.data(), c->send_cnt, 4 * (size_t)p, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int d = 0; d < p; ++d) C[c->dd_rank][d] = cnt[d];
    }
    for (mardyn_ctx* c : G->m) {
        mardyn_ctx* ctx = c;
        cudaStream_t s = c->stream;
        const int n = (int)c->n, b = c->cur;
        std::vector<int64_t> sc(p), rcap(p, 1);
        int64_t tot = 0;
        for (int d = 0; d < p; ++d) { sc[d] = std::max<int64_t>(C[c->dd_rank][d], 1); tot += sc[d]; }
        if (tot > c->seg_max * p) return fail(c, MARDYN_ECAPACITY, "rebalance: records exceed the send buffer");
        if (int rc = dd_set_segments(c, sc, rcap)) return rc;
        CK(cudaMemsetAsync(c->send_cnt, 0, sizeof(int) * p, s));
        DDArgs dd = dd_args(c, false);
        k_repartition<false><<<nblk(std::max(n, 1), 256), 256, 0, s>>>(n, c->g, dd, c->pos[b], c->vel[b],
                                                                        c->rigid ? c->quat[b] : nullptr,
                                                                        c->rigid ? c->angm[b] : nullptr,
                                                                        c->cell_of, c->rank, c->count);
        c->launches += 2;
        CK(cudaGetLastError());
    }
    if (int rc = gather_counts(G, C)) return rc;
    std::vector<int64_t> nrecv;
    if (int rc = exchange_exact(G, C, nrecv)) return rc;
    for (mardyn_ctx* c : G->m) {
        if (int rc = dd_import_sort(c, nrecv[c->dd_rank], false)) return rc;
        c->seg_ready = false;
        c->peer_segs = false;
        c->direct = false;
        c->last_rebalance = c->host_step;
        mardyn_ctx* ctx = c;
        int flag = 0;
        CK(cudaMemcpy(&flag, c->flag, 4, cudaMemcpyDeviceToHost));
        if (flag & 256) return fail(c, MARDYN_ECAPACITY, "rebalance: exchange segment overflow");
    }
    return MARDYN_OK;
}

// NVT (reading A24) on a decomposed run: after step k (k + 1 a multiple of the
// interval) the global KE of t_k (rank-ordered sum of the ranks' partials: ncclAllReduce, or
// read across the loopback ranks) sets lambda; every rank scales its molecules
static int group_thermostat(Group* G, long long k)
{
    mardyn_ctx* c0 = G->m[0];
    if (!(c0->T_target > 0) || c0->thermo_interval < 1 || (k + 1) % c0->thermo_interval != 0) return MARDYN_OK;
    const int p = G->p;
    std::vector<double*> ke;
    if (G->nccl) {
        mardyn_ctx* ctx = c0;
        double* d = reinterpret_cast<double*>(c0->cmat);
        k_ke_entry<<<1, 32, 0, c0->stream>>>(c0->hist, k, d);
        NCK(mdn::api().AllReduce(d, d, 2, ncclDouble, ncclSum, G->comm, c0->stream));
        c0->launches += 1;
        ke.push_back(d);
    } else {
        mardyn_ctx* ctx = c0;
        // the p history rings' addresses (after the two KE doubles of rank 0's scratch)
        double* d = reinterpret_cast<double*>(c0->cmat);
        const ObsRec** tab = reinterpret_cast<const ObsRec**>(c0->cmat + 2);
        G->hist_tab.resize(p);
        for (mardyn_ctx* c : G->m) G->hist_tab[c->dd_rank] = c->hist;
        CK(cudaMemcpyAsync(tab, G->hist_tab.data(), sizeof(void*) * p, cudaMemcpyHostToDevice, c0->stream));
        k_ke_sum<<<1, 32, 0, c0->stream>>>(p, tab, k, d);
        c0->launches += 1;
        for (int r = 0; r < p; ++r) ke.push_back(d);
    }
    for (size_t r = 0; r < G->m.size(); ++r) {
        mardyn_ctx* c = G->m[r];
        mardyn_ctx* ctx = c;
        k_rescale_global<<<std::min(nblk(c->cap, 256), 8 * c->num_sms), 256, 0, c->stream>>>(
            (int)c->cap, c->start + c->g.wncell, c->vel[c->cur], c->rigid ? c->angm[c->cur] : nullptr, ke[r],
            c->ndof_global, c->T_target, c->flag);
        c->launches += 1;
        CK(cudaGetLastError());
    }
    return MARDYN_OK;
}

// every rank of the group still exists (a destroyed loopback rank leaves a hole)
static bool group_ok(const Group* G)
{
    for (const mardyn_ctx* c : G->m)
        if (!c) return false;
    return true;
}

static int group_step(mardyn_ctx* ctx, int32_t nsteps)
{
    Group* G = ctx->grp;
    if (!G) return fail(ctx, MARDYN_ESTATE, "decomposed context without a group");
    if (!group_ok(G)) return fail(ctx, MARDYN_ESTATE, "a rank of the group was destroyed");
    if (!G->nccl && ctx != G->m[0]) return fail(ctx, MARDYN_ESTATE, "step a loopback group through its rank 0");
    for (mardyn_ctx* c : G->m) {
        if (c->poisoned) return fail(ctx, MARDYN_ECUDA, "a rank's context is poisoned");
        if (!c->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules on every rank first");
    }
    for (int k = 0; k < nsteps; ++k) {
        const long long st = ctx->host_step;
        if (ctx->rebalance_interval > 0 && st > 0 && st % ctx->rebalance_interval == 0 && ctx->last_rebalance != st) {
            if (int rc = group_rebalance(G)) return rc;
        }
        int rc = ctx->seg_ready ? group_async_step(G) : group_sync_step(G);
        if (rc) return rc;
        if ((rc = group_thermostat(G, st))) return rc;
    }
    for (mardyn_ctx* c : G->m) c->last_force_launches = nsteps;
    return MARDYN_OK;
}

static int group_compute_forces(mardyn_ctx* ctx)
{
    Group* G = ctx->grp;
    if (!group_ok(G)) return fail(ctx, MARDYN_ESTATE, "a rank of the group was destroyed");
    if (!G->nccl && ctx != G->m[0]) return fail(ctx, MARDYN_ESTATE, "compute_forces of a loopback group through rank 0");
    for (mardyn_ctx* c : G->m) {
        if (!c->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules on every rank first");
        if (int rc = compute_forces_local(c)) return rc;
    }
    return MARDYN_OK;
}

// global observable ring: per entry the rank-ordered sums (U, W, KE, pair and candidate
// counts; ranks count ordered pairs of their owned molecules) and T from the global N_dof
static int group_observables(mardyn_ctx* ctx, std::vector<ObsRec>& ring)
{
    NvtxRange nvtx_range("dd_observables");
    Group* G = ctx->grp;
    const int p = G->p;
    if (!group_ok(G)) return fail(ctx, MARDYN_ESTATE, "a rank of the group was destroyed");
    ring.assign(MD_HISTORY, ObsRec{});
    std::vector<ObsRec> h(MD_HISTORY * (size_t)p);
    if (G->nccl) {
        int rc = group_agree(G, sync_check(ctx));
        if (rc) return rc;
        NCK(mdn::api().AllGather(ctx->hist, ctx->obs_all, sizeof(ObsRec) * MD_HISTORY, ncclChar, G->comm, ctx->stream));
        CK(cudaMemcpyAsync(h.data(), ctx->obs_all, sizeof(ObsRec) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    } else {
        for (mardyn_ctx* c : G->m) {
            int rc = sync_check(c);
            if (rc) return fail(ctx, rc, c->err);
            CK(cudaMemcpy(h.data() + (size_t)c->dd_rank * MD_HISTORY, c->hist, sizeof(ObsRec) * MD_HISTORY,
                          cudaMemcpyDeviceToHost));
        }
    }
    for (int e = 0; e < MD_HISTORY; ++e) {
        ObsRec o = h[e];
        for (int r = 1; r < p; ++r) {
            const ObsRec& x = h[(size_t)r * MD_HISTORY + e];
            o.U += x.U; o.W += x.W; o.KEt += x.KEt; o.KEr += x.KEr; o.npairs += x.npairs; o.ncand += x.ncand;
        }
        if (ctx->nranks > 1) {
            o.npairs /= 2;
            o.T = 2.0 * (o.KEt + o.KEr) / ctx->ndof_global;
        }
        ring[e] = o;
    }
    return MARDYN_OK;
}

// ---- C ABI of the distributed engine

extern "C" {

int mardyn_nccl_unique_id(void* out128)
{
    if (!out128) return MARDYN_EINVAL;
    mdn::Api& A = mdn::api();
    if (!A.ok) return MARDYN_ENCCL;
    ncclUniqueId id;
    if (A.GetUniqueId(&id) != ncclSuccess) return MARDYN_ENCCL;
    std::memcpy(out128, &id, sizeof(id));
    return MARDYN_OK;
}

int mardyn_create_distributed(const double box[3], double cutoff, const mardyn_component* comps, int32_t n_comps,
                              const mardyn_options* opt, const void* nccl_unique_id, int32_t rank, int32_t world,
                              int32_t device, mardyn_ctx** out)
{
    if (!out) return MARDYN_EINVAL;
    *out = nullptr;
    if (!nccl_unique_id || world < 1 || world > 32 || rank < 0 || rank >= world) {
        mardyn_ctx* c = new mardyn_ctx();
        c->err = "bad rank / world (1..32) / unique id";
        *out = c;
        return MARDYN_EINVAL;
    }
    if (cudaSetDevice(device) != cudaSuccess) {
        mardyn_ctx* c = new mardyn_ctx();
        c->err = "cudaSetDevice failed";
        *out = c;
        return MARDYN_ECUDA;
    }
    int rc = mardyn_create(box, cutoff, comps, n_comps, opt, out);
    if (rc) return rc;
    mardyn_ctx* ctx = *out;
    mdn::Api& A = mdn::api();
    if (!A.ok) return fail(ctx, MARDYN_ENCCL, A.err);
    Group* G = new Group();
    G->p = world;
    G->nccl = true;
    G->m.push_back(ctx);
    G->live = 1;
    ctx->grp = G;
    ctx->nranks = world;
    ctx->dd_rank = rank;
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    NCK(A.CommInitRank(&G->comm, world, id, rank));
    if (world == 1) {                     // one rank: the single-domain step, observables through NCCL
        ctx->nranks = 1;
        std::vector<int32_t> b = {0, 0, 0, ctx->g.nc[0], ctx->g.nc[1], ctx->g.nc[2]};
        ctx->boxes = b;
    }
    return MARDYN_OK;
}

int mardyn_create_loopback(const double box[3], double cutoff, const mardyn_component* comps, int32_t n_comps,
                           const mardyn_options* opt, int32_t p, mardyn_ctx** out)
{
    if (!out || !opt || p < 2 || p > 32) return MARDYN_EINVAL;
    Group* G = new Group();
    G->p = p;
    mardyn_options o = *opt;
    if (!o.cuda_stream) {
        if (cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking) != cudaSuccess) { delete G; return MARDYN_ECUDA; }
        G->own_stream = true;
        o.cuda_stream = G->stream;
    } else {
        G->stream = (cudaStream_t)o.cuda_stream;
    }
    int rc = MARDYN_OK;
    for (int r = 0; r < p; ++r) {
        out[r] = nullptr;
        int e = mardyn_create(box, cutoff, comps, n_comps, &o, &out[r]);
        if (!out[r]) { rc = MARDYN_EINVAL; break; }
        out[r]->grp = G;
        out[r]->nranks = p;
        out[r]->dd_rank = r;
        G->m.push_back(out[r]);
        G->live += 1;
        if (e) { rc = e; break; }
    }
    if (G->live == 0) { if (G->own_stream) cudaStreamDestroy(G->stream); delete G; }
    return rc;
}

int mardyn_partition(mardyn_ctx* ctx, int64_t n, const double* r)
{
    if (!ctx || (n > 0 && !r) || n < 0) return MARDYN_EINVAL;
    if (ctx->nranks < 2) return MARDYN_OK;
    std::vector<int32_t> counts((size_t)ctx->g.ncell, 0);
    for (int64_t i = 0; i < n; ++i) counts[host_cell(ctx->g, r + 3 * i)] += 1;
    std::vector<int32_t> boxes;
    if (int rc = boxes_from_counts(ctx, counts.data(), boxes)) return rc;
    return dd_set_maps(ctx, boxes.data());
}

int mardyn_set_partition(mardyn_ctx* ctx, const int32_t* boxes)
{
    if (!ctx || !boxes) return MARDYN_EINVAL;
    if (ctx->nranks < 2) return fail(ctx, MARDYN_ESTATE, "not a decomposed context");
    if (ctx->loaded) ctx->loaded = false;       // the molecules must be loaded again
    group_drop_graphs(ctx->grp);
    return dd_set_maps(ctx, boxes);
}

int mardyn_get_partition(const mardyn_ctx* ctx, int32_t* boxes)
{
    if (!ctx || !boxes) return MARDYN_EINVAL;
    if (ctx->boxes.empty()) return MARDYN_ESTATE;
    std::memcpy(boxes, ctx->boxes.data(), sizeof(int32_t) * ctx->boxes.size());
    return MARDYN_OK;
}

int mardyn_dd_counts(mardyn_ctx* ctx, int64_t n, const double* r, int64_t* counts)
{
    if (!ctx || !counts || (n > 0 && !r) || n < 0) return MARDYN_EINVAL;
    const int p = ctx->nranks;
    if (p < 2) { counts[0] = n; return MARDYN_OK; }
    if (ctx->h_owner.empty()) return fail(ctx, MARDYN_ESTATE, "mardyn_partition first");
    for (int q = 0; q < p; ++q) counts[q] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t c = host_cell(ctx->g, r + 3 * i);
        counts[ctx->h_owner[c]] += 1;
        for (uint32_t m = ctx->h_gmask[c]; m; m &= m - 1) counts[__builtin_ctz(m)] += 1;
    }
    return MARDYN_OK;
}

// host-only helpers (no context, no GPU): the lattice and cells of reading A12 and the k-d
// partition of a set of positions -- the functions mardyn_partition and the rebalance use
int mardyn_grid_counts(const double box[3], double cutoff, int64_t n, const double* r, int32_t ncell[3],
                       int32_t* counts)
{
    if (!box || !ncell || n < 0 || (n > 0 && !r) || !(cutoff > 0)) return MARDYN_EINVAL;
    GridP g;
    std::string err;
    if (int rc = grid_setup(box, cutoff, 1.0, g, err)) return rc;
    for (int k = 0; k < 3; ++k) ncell[k] = g.nc[k];
    if (!counts) return MARDYN_OK;
    std::fill(counts, counts + g.ncell, 0);
    for (int64_t i = 0; i < n; ++i) counts[host_cell(g, r + 3 * i)] += 1;
    return MARDYN_OK;
}

int mardyn_kd_partition(const double box[3], double cutoff, int64_t n, const double* r, int32_t p, int32_t* boxes,
                        double* loads)
{
    if (!boxes || p < 1) return MARDYN_EINVAL;
    int32_t nc[3];
    if (int rc = mardyn_grid_counts(box, cutoff, n, r, nc, nullptr)) return rc;
    std::vector<int32_t> counts((size_t)nc[0] * nc[1] * nc[2]);
    mardyn_grid_counts(box, cutoff, n, r, nc, counts.data());
    std::vector<double> cost(counts.size());
    mdd::cell_cost(counts.data(), nc[0], nc[1], nc[2], cost.data());
    return mardyn_kd_decompose(cost.data(), nc[0], nc[1], nc[2], p, boxes, loads);
}

int mardyn_set_cost_model(mardyn_ctx* ctx, int32_t model)
{
    if (!ctx) return MARDYN_EINVAL;
    if (model != 0 && model != 1) return fail(ctx, MARDYN_EINVAL, "cost model: 0 = Eq. 6, 1 = molecule count");
    for (mardyn_ctx* c : group_members(ctx)) c->cost_model = model;
    return MARDYN_OK;
}

int mardyn_rebalance(mardyn_ctx* ctx)
{
    if (!ctx) return MARDYN_EINVAL;
    if (ctx->nranks < 2 || !ctx->grp) return MARDYN_OK;
    Group* G = ctx->grp;
    if (!group_ok(G)) return fail(ctx, MARDYN_ESTATE, "a rank of the group was destroyed");
    if (!G->nccl && ctx != G->m[0]) return fail(ctx, MARDYN_ESTATE, "rebalance a loopback group through its rank 0");
    for (mardyn_ctx* c : G->m)
        if (!c->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules on every rank first");
    return group_rebalance(G);
}

}  // extern "C"
