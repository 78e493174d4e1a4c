// kprof.cpp -- per-kernel-class timing with CUDA events on the launching
// stream (bench.py's live roofline measurement).
#include <cstring>

#include <cstdio>
#include <cstdlib>

#include "hs_internal.h"

KTimer::KTimer(hs_ctx *c_, int id_, double bytes_, cudaStream_t st_) : c(c_), id(id_), bytes(bytes_), st(st_), slot(-1)
{
    if (!c->kprof_on) return;
    if (c->kprof_used * 2 + 2 > c->kprof_ev.size()) {
        size_t old = c->kprof_ev.size();
        c->kprof_ev.resize(old ? old * 2 : 4096);
        for (size_t i = old; i < c->kprof_ev.size(); i++) cudaEventCreate(&c->kprof_ev[i]);
        c->kprof_id.resize(c->kprof_ev.size() / 2);
        c->kprof_bytes.resize(c->kprof_ev.size() / 2);
    }
    slot = (int)c->kprof_used++;
    c->kprof_id[slot] = id;
    c->kprof_bytes[slot] = bytes;
    // under stream capture an External record becomes an event-record node of
    // the graph (a plain record would only express a dependency)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    ext = cs != cudaStreamCaptureStatusNone;
    if (ext) cudaEventRecordWithFlags(c->kprof_ev[2 * slot], st, cudaEventRecordExternal);
    else cudaEventRecord(c->kprof_ev[2 * slot], st);
}

KTimer::~KTimer()
{
    if (slot < 0) return;
    if (ext) cudaEventRecordWithFlags(c->kprof_ev[2 * slot + 1], st, cudaEventRecordExternal);
    else cudaEventRecord(c->kprof_ev[2 * slot + 1], st);
}

extern "C" {

hs_status hs_kprof_enable(hs_ctx *c, int on)
{
    if (!c) return HS_EINVAL;
    // switching on starts a new recording; switching off keeps the recorded
    // slots (a plan captured while on replays into them)
    if (on && !c->kprof_on) c->kprof_used = 0;
    c->kprof_on = on != 0;
    return HS_OK;
}

// out: per kernel class [launches, total ms, total algorithmic bytes] (KID_COUNT x 3)
hs_status hs_kprof_collect(hs_ctx *c, double *out, int n_classes)
{
    if (!c || !out) return HS_EINVAL;
    cudaDeviceSynchronize();
    memset(out, 0, sizeof(double) * 3 * n_classes);
    // dev diagnostic: HS_KPROF_DUMP=path appends one "class,bytes,ms" line per launch
    const char *dump = getenv("HS_KPROF_DUMP");
    FILE *fh = dump ? fopen(dump, "a") : nullptr;
    for (size_t i = 0; i < c->kprof_used; i++) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->kprof_ev[2 * i], c->kprof_ev[2 * i + 1]);
        int id = c->kprof_id[i];
        if (fh) fprintf(fh, "%d,%.0f,%.6f\n", id, c->kprof_bytes[i], ms);
        if (id >= n_classes) continue;
        out[3 * id] += 1;
        out[3 * id + 1] += ms;
        out[3 * id + 2] += c->kprof_bytes[i];
    }
    if (fh) fclose(fh);
    c->kprof_used = 0;
    return HS_OK;
}

}
