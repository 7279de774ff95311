// capi_ext.cu -- the C ABI, continued (same translation unit as capi.cu, whose
// helpers it uses): streaming encode / decode with a device carry (stream.cu),
// the one-sided cross-GPU error combine (peer.cu) and the overlapped
// host-buffer pipelines.  See include/b64gpu.h for every entry point's contract.

extern "C" {
// ---------------------------------------------------------------- streaming (stream.cu)
// The host side of a stream only does length arithmetic (held / consumed /
// produced are functions of the piece lengths), so no call waits for the
// device; the held bytes themselves live in the caller's device carry buffer.
namespace {
enum { kStIdle = 0, kStEncode = 1, kStDecode = 2, kStDone = 3 };
constexpr int32_t kStOverlap = 0x100;  // state bit: B64_STREAM_OVERLAP
inline int32_t st_kind(const b64_stream* st) { return st->state & 0xff; }
}

int64_t b64_stream_update_len(const b64_stream* st, int64_t len) {
    if (!st || len < 0) return -1;
    const int64_t A = st->held + len;
    if (st_kind(st) == kStEncode) return 4 * (A / 3);                 // whole triples
    if (st_kind(st) == kStDecode) return A > 0 ? 3 * ((A - 1) / 4) : 0;  // the last 1..4 chars are held
    return -1;
}

int64_t b64_stream_end_len(const b64_stream* st) {
    if (!st) return -1;
    if (st_kind(st) == kStEncode) return st->held > 0 ? 4 : 0;  // the padded tail
    if (st_kind(st) == kStDecode) return (st->consumed > 0 && st->consumed % 4 == 0) ? 3 : 0;
    return -1;
}

int b64_encode_stream_begin(b64_stream* st, uint8_t* d_carry) {
    if (!st || !d_carry) return B64_EINVAL;
    st->consumed = st->produced = 0;
    st->held = 0;
    st->state = kStEncode;
    st->d_carry = d_carry;
    st->d_err_min = nullptr;
    return B64_OK;
}

int b64_encode_stream_begin_ex(b64_stream* st, uint8_t* d_carry, uint32_t flags, b64_stream_t stream) {
    if (!st || !d_carry || (flags & ~B64_STREAM_OVERLAP)) return B64_EINVAL;
    if (flags & B64_STREAM_OVERLAP) {
        // a memset, not a kernel: the first piece is fully ordered after everything before the
        // begin call (no programmatic edge crosses it), which the overlap mode relies on
        if (cudaMemsetAsync(d_carry, 0, 8, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess) return B64_ECUDA;
    }
    const int r = b64_encode_stream_begin(st, d_carry);
    if (r == B64_OK && (flags & B64_STREAM_OVERLAP)) st->state |= kStOverlap;
    return r;
}

int b64_encode_stream_update(b64_stream* st, const uint8_t* d_in, int64_t n, uint8_t* d_out, const b64_alphabet* a,
                             int64_t* n_out, b64_stream_t stream) {
    if (!st || st_kind(st) != kStEncode || n < 0 || !alpha_ok(a) || (n > 0 && !d_in)) return B64_EINVAL;
    const int64_t H = st->held, A = H + n, T = A / 3;
    if (T > 0 && !d_out) return B64_EINVAL;
    if (n_out) *n_out = 4 * T;
    if (n == 0) return B64_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int join = (H > 0 && T > 0) ? 1 : 0;
    const int64_t skip = join ? 3 - H : 0, tb = T - join;  // whole triples read straight from the piece
    if ((st->state & kStOverlap) && st->consumed > 0 && 3 * tb >= unaligned_min() &&
        aligned(d_out + 4 * join, 4)) {
        // overlap mode (B64_STREAM_OVERLAP), from the second piece on: the bulk runs while the
        // previous piece drains, the join (reading the carry it writes) at its end, after the wait
        const EncJoin ej = {st->d_carry, d_in, d_out, n, int32_t(H), (H > 0 || A % 3) ? 1 : 0};
        const int r = encode_launch(d_in + skip, 3 * tb, d_out + 4 * join, a, s, true, &ej);
        if (r != B64_OK) return r;
        st->held = int32_t(A % 3);
        st->consumed += n;
        st->produced += 4 * T;
        return B64_OK;
    }
    if (H > 0 || A % 3) {  // a straddling triple and / or bytes to hold: one thread, before the bulk
        // (riding along with enc_fastu_kernel, first or last thread, measured 4 % slower on
        // 64 MiB pieces: its dependent loads sit on the piece's critical path)
        launch(enc_stream_join_kernel, 1, 1, s, st->d_carry, int(H), d_in, n, d_out, enc_tab(a));
        const int r = launched();
        if (r != B64_OK) return r;
    }
    if (tb > 0) {
        const int r = encode_launch(d_in + skip, 3 * tb, d_out + 4 * join, a, s);
        if (r != B64_OK) return r;
    }
    st->held = int32_t(A % 3);
    st->consumed += n;
    st->produced += 4 * T;
    return B64_OK;
}

int b64_encode_stream_end(b64_stream* st, uint8_t* d_out, const b64_alphabet* a, int64_t* n_out,
                          b64_stream_t stream) {
    if (!st || st_kind(st) != kStEncode || !alpha_ok(a)) return B64_EINVAL;
    const int H = st->held;
    if (H > 0 && !d_out) return B64_EINVAL;
    if (n_out) *n_out = H > 0 ? 4 : 0;
    if (H > 0) {
        launch(enc_stream_end_kernel, 1, 1, reinterpret_cast<cudaStream_t>(stream), st->d_carry, H, d_out, enc_tab(a),
               uint32_t(a->pad));
        const int r = launched();
        if (r != B64_OK) return r;
        st->produced += 4;
    }
    st->held = 0;
    st->state = kStDone;
    return B64_OK;
}

int b64_decode_stream_begin_ex(b64_stream* st, uint8_t* d_carry, int64_t* d_err_min, uint32_t flags,
                                b64_stream_t stream) {
    if (!st || !d_carry || !d_err_min || (flags & ~B64_STREAM_OVERLAP)) return B64_EINVAL;
    // a memset, not a kernel: the first piece is fully ordered after everything before the begin
    // call (no programmatic edge crosses it), which the overlap mode relies on
    if (cudaMemsetAsync(d_err_min, 0x7F, sizeof(int64_t), reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess)
        return B64_ECUDA;
    st->consumed = st->produced = 0;
    st->held = 0;
    st->state = kStDecode | ((flags & B64_STREAM_OVERLAP) ? kStOverlap : 0);
    st->d_carry = d_carry;
    st->d_err_min = d_err_min;
    return B64_OK;
}

int b64_decode_stream_begin(b64_stream* st, uint8_t* d_carry, int64_t* d_err_min, b64_stream_t stream) {
    return b64_decode_stream_begin_ex(st, d_carry, d_err_min, 0u, stream);
}

int b64_decode_stream_update(b64_stream* st, const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a,
                             int64_t* n_out, b64_stream_t stream) {
    if (!st || st_kind(st) != kStDecode || m < 0 || !alpha_ok(a) || (m > 0 && !d_in)) return B64_EINVAL;
    const int64_t H = st->held, A = H + m;
    const int64_t Q = A > 0 ? (A - 1) / 4 : 0;  // the last 1..4 chars are always held
    if (Q > 0 && !d_out) return B64_EINVAL;
    if (n_out) *n_out = 3 * Q;
    if (m == 0) return B64_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int join = (H > 0 && Q > 0) ? 1 : 0;
    const int64_t skip = join ? 4 - H : 0, qb = Q - join;  // whole quads read straight from the piece
    // the join (held chars + the piece's head, and the new carry) rides along with the piece's
    // bulk kernel when that is the fast one; otherwise it is a one-thread kernel of its own
    // overlap mode (B64_STREAM_OVERLAP): from the second piece on, the bulk runs before
    // griddepcontrol.wait, i.e. while the previous piece's kernel drains (R15)
    const bool early = (st->state & kStOverlap) && st->consumed > 0;
    const StreamJoin sj = {st->d_carry, d_in, d_out, m, st->consumed - H, int32_t(H), 1};
    bool joined = false;
    int r = B64_OK;
    if (qb > 0) {
        r = decode_launch(d_in + skip, 4 * qb, d_out + 3 * join, a, st->consumed + skip, 0, st->d_err_min, nullptr,
                          s, &sj, &joined, early);
        if (r != B64_OK) return r;
    }
    if (!joined) {
        launch(dec_stream_join_kernel, 1, 1, s, st->d_carry, int(H), d_in, m, d_out, dec_tab(a), st->consumed - H,
               reinterpret_cast<unsigned long long*>(st->d_err_min));
        r = launched();
        if (r != B64_OK) return r;
    }
    st->held = int32_t(A - 4 * Q);
    st->consumed += m;
    st->produced += 3 * Q;
    return B64_OK;
}

int b64_decode_stream_end(b64_stream* st, uint8_t* d_out, const b64_alphabet* a, int64_t* d_err_off,
                          int32_t* d_status, int64_t* d_out_len, int64_t* n_out, b64_stream_t stream) {
    if (!st || st_kind(st) != kStDecode || !alpha_ok(a) || !d_err_off) return B64_EINVAL;
    const int64_t total = st->consumed;
    const bool fin = total > 0 && total % 4 == 0;
    if (fin && !d_out) return B64_EINVAL;
    launch(dec_stream_end_kernel, 1, 1, reinterpret_cast<cudaStream_t>(stream), st->d_carry, int(st->held), total,
           d_out, dec_tab(a), reinterpret_cast<const unsigned long long*>(st->d_err_min), d_err_off, d_status,
           d_out_len);
    const int r = launched();
    if (r != B64_OK) return r;
    if (n_out) *n_out = fin ? 3 : 0;  // bytes of d_out the end call may write (the exact count is in *d_out_len)
    st->held = 0;
    st->state = kStDone;
    return B64_OK;
}

// ---------------------------------------------------------------- one-sided peer combine (peer.cu)
int64_t b64_peer_combine_bytes(int64_t count) {
    return count < 0 ? -1 : std::max<int64_t>(64, 2ll * kPeerMaxWorld * count * 16);
}

int b64_peer_combine_init(uint8_t* d_buf, int64_t count, b64_stream_t stream) {
    if (!d_buf || count < 0) return B64_EINVAL;
    launch(peer_buffer_init_kernel, 1, kThreads, reinterpret_cast<cudaStream_t>(stream), d_buf, count);
    return launched();
}

int b64_peer_combine(uint8_t* const* d_bufs, int world, int rank, const int64_t* d_local, int64_t count,
                     uint64_t epoch, int64_t* d_err_off, int32_t* d_status, b64_stream_t stream) {
    if (!d_bufs || world < 1 || world > 32 || rank < 0 || rank >= world || count < 0 || count > 4096 ||
        (count > 0 && (!d_local || !d_err_off)))
        return B64_EINVAL;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = size_t(count) * 8;
    cfg.stream = reinterpret_cast<cudaStream_t>(stream);
    note(cudaLaunchKernelEx(&cfg, peer_combine_kernel, d_bufs, world, rank,
                            reinterpret_cast<const unsigned long long*>(d_local), count,
                            static_cast<unsigned long long>(epoch), d_err_off, d_status));
    return launched();
}

int b64_peer_buffer_alloc(int64_t bytes, uint8_t** d_buf, uint8_t handle[64]) {
    if (bytes <= 0 || !d_buf || !handle) return B64_EINVAL;
    void* p = nullptr;
    if (cudaMalloc(&p, size_t(bytes)) != cudaSuccess) return (cudaGetLastError(), B64_ECUDA);
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return (cudaGetLastError(), B64_ECUDA);
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
    *d_buf = static_cast<uint8_t*>(p);
    return B64_OK;
}

int b64_peer_buffer_open(const uint8_t handle[64], uint8_t** d_buf) {
    if (!handle || !d_buf) return B64_EINVAL;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return (cudaGetLastError(), B64_ECUDA);
    *d_buf = static_cast<uint8_t*>(p);
    return B64_OK;
}

int b64_peer_buffer_release(uint8_t* d_buf, int opened) {
    if (!d_buf) return B64_EINVAL;
    const cudaError_t e = opened ? cudaIpcCloseMemHandle(d_buf) : cudaFree(d_buf);
    return e == cudaSuccess ? B64_OK : (cudaGetLastError(), B64_ECUDA);
}

int b64_peer_combine_emulate(uint8_t* const* d_bufs, int world, const int64_t* d_local, int64_t count, int epochs,
                             int64_t* d_out, int* d_ok, b64_stream_t stream) {
    if (!d_bufs || world < 1 || world > 32 || count < 0 || epochs < 0 || !d_ok || (count > 0 && (!d_local || !d_out)))
        return B64_EINVAL;
    uint8_t* const* b = d_bufs;
    int w = world;
    const unsigned long long* l = reinterpret_cast<const unsigned long long*>(d_local);
    int64_t k = count;
    int e = epochs;
    unsigned long long* o = reinterpret_cast<unsigned long long*>(d_out);
    int* okp = d_ok;
    void* args[] = {&b, &w, &l, &k, &e, &o, &okp};
    // all `world` blocks wait on one another: a cooperative launch guarantees they are co-resident
    note(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(peer_combine_emulate_kernel), dim3(world), dim3(32),
                                     args, 0, reinterpret_cast<cudaStream_t>(stream)));
    return launched();
}

// ---------------------------------------------------------------- host-buffer pipelines
// Chunks of the host input are copied H2D on s_h2d, coded on s_comp and copied
// back D2H on s_d2h through kHostBufs rotating device buffers, so both PCIe
// directions and the kernels overlap.  Cross-stream order uses events created
// for the call and released at its end (the library keeps no state).
namespace {
constexpr int kHostBufs = 3;

struct HostPipe {
    cudaEvent_t h2d[kHostBufs], comp[kHostBufs], d2h[kHostBufs];
    bool ok = true;
    HostPipe() {
        for (int i = 0; i < kHostBufs; ++i) {
            ok &= cudaEventCreateWithFlags(&h2d[i], cudaEventDisableTiming) == cudaSuccess;
            ok &= cudaEventCreateWithFlags(&comp[i], cudaEventDisableTiming) == cudaSuccess;
            ok &= cudaEventCreateWithFlags(&d2h[i], cudaEventDisableTiming) == cudaSuccess;
        }
    }
    // The workspace buffers may still be in use by work already queued on the
    // three streams (a previous call): the first copy of this call waits for it.
    cudaError_t order_after_previous(cudaStream_t sh, cudaStream_t sc, cudaStream_t sd) {
        cudaError_t e = cudaEventRecord(comp[0], sc);
        if (e == cudaSuccess) e = cudaEventRecord(d2h[0], sd);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sh, comp[0], 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sh, d2h[0], 0);
        return e;
    }
    ~HostPipe() {
        for (int i = 0; i < kHostBufs; ++i) {
            cudaEventDestroy(h2d[i]);
            cudaEventDestroy(comp[i]);
            cudaEventDestroy(d2h[i]);
        }
    }
};

int64_t align_down(int64_t v, int64_t a) { return v / a * a; }
}  // namespace

int64_t b64_host_workspace_bytes(int64_t chunk_bytes) {
    if (chunk_bytes <= 0) return -1;
    const int64_t c = align_down(chunk_bytes, 3072) > 0 ? align_down(chunk_bytes, 3072) : 3072;
    return kHostBufs * (c + (c / 3) * 4 + 512) + 256;
}

int b64_encode_host(const uint8_t* h_in, int64_t n, uint8_t* h_out, const b64_alphabet* a, uint8_t* d_ws,
                    int64_t ws_bytes, b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h) {
    return b64_encode_host_ex(h_in, n, h_out, a, d_ws, ws_bytes, s_h2d, s_comp, s_d2h, 0u);
}

// One chunk's hand-over between the three streams: every runtime call checked.
#define B64_CK(call)                                  \
    do {                                              \
        if ((call) != cudaSuccess) {                  \
            cudaGetLastError();                       \
            return B64_ECUDA;                         \
        }                                             \
    } while (0)

int b64_encode_host_ex(const uint8_t* h_in, int64_t n, uint8_t* h_out, const b64_alphabet* a, uint8_t* d_ws,
                       int64_t ws_bytes, b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h,
                       unsigned flags) {
    if (n < 0 || !alpha_ok(a) || (flags & ~unsigned(B64_HOST_CALLER_ORDERED))) return B64_EINVAL;
    if (n == 0) return B64_OK;
    if (!h_in || !h_out || !d_ws) return B64_EINVAL;
    // per buffer: C input bytes + 4C/3 output chars; C a multiple of 3072 (= 4 * 768, keeps both aligned)
    const int64_t per = (ws_bytes - 256) / kHostBufs - 512;
    const int64_t C = align_down(per * 3 / 7, 3072);
    if (C <= 0) return B64_EINVAL;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(d_ws) + 255) & ~uintptr_t(255));
    cudaStream_t sh = reinterpret_cast<cudaStream_t>(s_h2d), sc = reinterpret_cast<cudaStream_t>(s_comp),
                 sd = reinterpret_cast<cudaStream_t>(s_d2h);
    HostPipe pipe;
    if (!pipe.ok) return B64_ECUDA;
    if (!(flags & B64_HOST_CALLER_ORDERED)) B64_CK(pipe.order_after_previous(sh, sc, sd));
    const int64_t stride = C + C / 3 * 4 + 512;
    int64_t j = 0;
    for (int64_t off = 0; off < n; off += C, ++j) {
        const int b = int(j % kHostBufs);
        uint8_t* din = base + b * stride;
        uint8_t* dout = din + C + 256;
        const int64_t len = (n - off < C) ? n - off : C;
        const int64_t olen = b64_encoded_len(len);
        if (j >= kHostBufs) B64_CK(cudaStreamWaitEvent(sh, pipe.d2h[b], 0));
        B64_CK(cudaMemcpyAsync(din, h_in + off, size_t(len), cudaMemcpyHostToDevice, sh));
        B64_CK(cudaEventRecord(pipe.h2d[b], sh));
        B64_CK(cudaStreamWaitEvent(sc, pipe.h2d[b], 0));
        const int r = b64_encode(din, len, dout, a, s_comp);
        if (r != B64_OK) return r;
        B64_CK(cudaEventRecord(pipe.comp[b], sc));
        B64_CK(cudaStreamWaitEvent(sd, pipe.comp[b], 0));
        B64_CK(cudaMemcpyAsync(h_out + off / 3 * 4, dout, size_t(olen), cudaMemcpyDeviceToHost, sd));
        B64_CK(cudaEventRecord(pipe.d2h[b], sd));
    }
    return B64_OK;
}

int b64_decode_host(const uint8_t* h_in, int64_t m, uint8_t* h_out, const b64_alphabet* a, uint8_t* d_ws,
                    int64_t ws_bytes, int64_t* d_err_off, int32_t* d_status, int64_t* d_out_len, b64_stream_t s_h2d,
                    b64_stream_t s_comp, b64_stream_t s_d2h) {
    return b64_decode_host_ex(h_in, m, h_out, a, d_ws, ws_bytes, d_err_off, d_status, d_out_len, s_h2d, s_comp, s_d2h,
                              0u);
}

int b64_decode_host_ex(const uint8_t* h_in, int64_t m, uint8_t* h_out, const b64_alphabet* a, uint8_t* d_ws,
                       int64_t ws_bytes, int64_t* d_err_off, int32_t* d_status, int64_t* d_out_len,
                       b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h, unsigned flags) {
    if (m < 0 || !alpha_ok(a) || !d_err_off || (flags & ~unsigned(B64_HOST_CALLER_ORDERED))) return B64_EINVAL;
    if (m % 4) return B64_ELENGTH;
    if (m > 0 && (!h_in || !h_out || !d_ws)) return B64_EINVAL;
    cudaStream_t sh = reinterpret_cast<cudaStream_t>(s_h2d), sc = reinterpret_cast<cudaStream_t>(s_comp),
                 sd = reinterpret_cast<cudaStream_t>(s_d2h);
    B64_CK(cudaMemsetAsync(d_err_off, 0x7F, sizeof(int64_t), sc));
    if (m == 0) {
        if (d_out_len) B64_CK(cudaMemsetAsync(d_out_len, 0, sizeof(int64_t), sc));
        return b64_decode_finalize(d_err_off, d_err_off, d_status, s_comp);
    }
    // per buffer: C chars + 3C/4 bytes; C a multiple of 4096 (= 4 * 1024)
    const int64_t per = (ws_bytes - 256) / kHostBufs - 512;
    const int64_t C = align_down(per * 4 / 7, 4096);
    if (C <= 0) return B64_EINVAL;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(d_ws) + 255) & ~uintptr_t(255));
    HostPipe pipe;
    if (!pipe.ok) return B64_ECUDA;
    if (!(flags & B64_HOST_CALLER_ORDERED)) B64_CK(pipe.order_after_previous(sh, sc, sd));
    const int64_t stride = C + C / 4 * 3 + 512;
    int64_t j = 0, last_off = 0;
    for (int64_t off = 0; off < m; off += C, ++j) {
        const int b = int(j % kHostBufs);
        uint8_t* din = base + b * stride;
        uint8_t* dout = din + C + 256;
        const int64_t len = (m - off < C) ? m - off : C;
        const bool fin = off + len == m;
        if (j >= kHostBufs) B64_CK(cudaStreamWaitEvent(sh, pipe.d2h[b], 0));
        B64_CK(cudaMemcpyAsync(din, h_in + off, size_t(len), cudaMemcpyHostToDevice, sh));
        B64_CK(cudaEventRecord(pipe.h2d[b], sh));
        B64_CK(cudaStreamWaitEvent(sc, pipe.h2d[b], 0));
        // the final chunk also reports its valid-text length (pads subtracted, on the device)
        const int r = b64_decode_chunk(din, len, dout, a, off, fin ? 1 : 0, d_err_off, fin ? d_out_len : nullptr,
                                       s_comp);
        if (r != B64_OK) return r;
        B64_CK(cudaEventRecord(pipe.comp[b], sc));
        B64_CK(cudaStreamWaitEvent(sd, pipe.comp[b], 0));
        B64_CK(cudaMemcpyAsync(h_out + off / 4 * 3, dout, size_t(len / 4 * 3), cudaMemcpyDeviceToHost, sd));
        B64_CK(cudaEventRecord(pipe.d2h[b], sd));
        last_off = off;
    }
    // packed error word -> (err_off, status) and the exact output length: the final chunk's
    // valid length plus the bytes of the chunks before it, or 3*floor(err/4) on an error
    launch(dec_finalize_len_kernel, 1, 1, sc, static_cast<const int64_t*>(d_err_off), d_err_off, d_status, d_out_len,
           last_off / 4 * 3);
    return launched();
}
#undef B64_CK

// ---------------------------------------------------------------- decode -> consumer (f3)
int64_t b64_consume_chunk_chars(int64_t ring_bytes) {
    if (ring_bytes < 3072) return -1;
    return ring_bytes / 3 * 4 / 4096 * 4096;  // 3C/4 decoded bytes fit the ring; C % 4096 == 0
}

int b64_decode_consume(const uint8_t* d_in, int64_t m, uint8_t* d_ring, int64_t ring_bytes, const b64_alphabet* a,
                       b64_consumer_fn consumer, void* user, int64_t* d_err_off, int32_t* d_status,
                       int64_t* d_out_len, b64_stream_t stream) {
    if (m < 0 || !alpha_ok(a) || !d_err_off || !consumer) return B64_EINVAL;
    if (m % 4) return B64_ELENGTH;
    if (m > 0 && (!d_in || !d_ring)) return B64_EINVAL;
    const int64_t C = b64_consume_chunk_chars(ring_bytes);
    if (m > 0 && C <= 0) return B64_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    note(cudaMemsetAsync(d_err_off, 0x7F, sizeof(int64_t), s));
    if (m == 0) {
        if (d_out_len) note(cudaMemsetAsync(d_out_len, 0, sizeof(int64_t), s));
        int r = launched();
        if (r != B64_OK) return r;
        g_launches.fetch_sub(1, std::memory_order_relaxed);  // memsets, not kernels
        return b64_decode_finalize(d_err_off, d_err_off, d_status, stream);
    }
    int64_t last_off = 0;
    for (int64_t off = 0; off < m; off += C) {
        const int64_t len = (m - off < C) ? m - off : C;
        const bool fin = off + len == m;
        const int r = b64_decode_chunk(d_in + off, len, d_ring, a, off, fin ? 1 : 0, d_err_off,
                                       fin ? d_out_len : nullptr, stream);
        if (r != B64_OK) return r;
        consumer(d_ring, len / 4 * 3, off / 4 * 3, user, stream);  // reads the chunk while it is in L2
        last_off = off;
    }
    launch(dec_finalize_len_kernel, 1, 1, s, static_cast<const int64_t*>(d_err_off), d_err_off, d_status, d_out_len,
           last_off / 4 * 3);
    return launched();
}

}  // extern "C"
