"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

O7: continuous-batching replay of one decode iteration per step
(SURVEY.md §8(a) S1 -> S7), driven by step latencies logged from the GPU run.

The paper describes the control loop only at the level of Fig. 1 / Alg. 1-2:
b_t is decided per scheduling interval from telemetry and bounds the number of
requests in the running batch.  The step semantics
below are the readings R17-R22 of DESIGN.md (SPEC.md:381-404 engine, adapted
to paged blocks):

 1. release arrivals with arrival_ns <= clock into the FCFS queue;
 2. admission: while the queue is non-empty and |running| < b_t (this rank's
    share of b_t), take the head r; it needs ceil((T_r + 1) / P) free pages
    with T_r = l_in + generated_r (recompute after preemption); otherwise
    stop (head-of-line blocking).  Admitted: append T_r tokens (prefill);
 3. page growth: every running request appends its decode token; while the
    pages this needs exceed the free pages, preempt the most recently admitted
    running request (LIFO; its pages are released, it goes to the queue head,
    its generated tokens are kept for recompute); then append (all-or-nothing);
 4. decode: the running requests in admission order attend over ctx_i tokens;
    the batch statistics record is formed (O3);
 5. retire requests with generated = l_out (release pages);
 6. clock += step_ns (device-timed); release arrivals; N^p = queue length;
 7. b_{t+1} from the scheduler on the (global) record (O5/O6).
An idle engine (nothing running or queued) jumps the clock to the next arrival.

PD fusion ("our method is also valid for determining
chunk size"; readings R25-R28 of DESIGN.md): prefill shares the iteration.
Admitted requests first PREFILL in chunks, then decode.  Step order (replaces 2-3):
 a. decode growth of the running (fully prefilled) requests, LIFO preemption over the
    admission order running ++ prefilling (a victim's prefill progress is discarded);
 b. chunk budget c_t = max(0, min(b_share, max_rows) - N^d), N^d = |running| (R25); with a
    fixed iteration token budget B (R36): c_t = max(0, min(B, max_rows) - N^d) while b_share
    still bounds |running| + |prefilling| in step c;
 c. FCFS chunk: prefilling requests in admission order, then new admissions from the queue
    head (while |running| + |prefilling| < b_share and the whole prompt + 1 fits the free
    pages, head-of-line blocking), each taking min(remaining prompt, budget left) tokens;
    an in-progress prefill is cut to the pages that are free (and the chunk stops there);
 d. attention: decode over the running batch, causal prefill attention over each chunk;
 e. requests whose prompt is complete join the running batch at the END of the step (they
    emit their first token in the next step).
N^p (n_waiting) = released requests not in this step's decode batch = queue + prefilling.

Swap preemption ("temporarily moving data from GPU memory
to CPU memory when capacity is exceeded.  The data are moved back to the GPU when space
becomes available"; readings R29-R31 of DESIGN.md), non-PD steps only:
 3'. a victim of step 3 whose pages fit the free swap pages (swap_cap_pages in total) is
     swapped out: its device pages are released exactly as on recompute and it goes to the
     queue head, but it keeps its KV (ctx = l_in + generated) in swap pages; otherwise it is
     preempted for recompute as before;
 2'. admitting a swapped-out head needs the same ceil((T + 1) / P) free pages; it gets
     ceil(T / P) pages lowest-free-first (the pages a prefill of T tokens would take) and its
     swap pages are freed -- the page tables are identical to recompute; only the KV's origin
     (copied back instead of recomputed) and the step latency differ.
"""
from __future__ import annotations

from collections import deque

from . import stats as ostats
from .allocator import PagedKV
from .policy import Scheduler

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
M64 = (1 << 64) - 1


def fnv1a64(values, h=FNV_OFFSET):
    """FNV-1a over 64-bit words, h = (h ^ v) * prime mod 2^64 (checksum of block tables)."""
    for v in values:
        h = ((h ^ (v & M64)) * FNV_PRIME) & M64
    return h


class RankEngine:
    """One GPU's request shard (DP) or the whole batch (G = 1 / TP)."""

    def __init__(self, req_ids, arrival_ns, l_in, l_out, cap_pages, page_size, rank=0, world=1,
                 pd=False, max_rows=None, swap_cap_pages=0, pd_token_budget=0):
        self.pd = bool(pd)
        self.pd_token_budget = int(pd_token_budget)  # R36: fixed iteration token budget (0: R25, b_t)
        if swap_cap_pages and pd:
            raise ValueError("swap preemption is defined for non-PD steps only")
        self.swap_cap = int(swap_cap_pages)  # 0: recompute only
        self.swapped = {}                    # request -> swap pages held
        self.swap_used = 0
        self.last_swaps = (0, 0)             # (swapped out, swapped in) of the last step
        self.max_rows = max_rows
        self.prefilling = []          # PD: [req, prompt tokens done], admission order
        self.last_chunks = []         # PD: (req, q_start, q_len) of the last step
        self.req_ids = list(req_ids)
        self.arrival = [int(a) for a in arrival_ns]
        self.l_in = {r: int(x) for r, x in zip(self.req_ids, l_in)}
        self.l_out = {r: int(x) for r, x in zip(self.req_ids, l_out)}
        self.kv = PagedKV(cap_pages, page_size)
        self.P = page_size
        self.cap = cap_pages
        self.rank, self.world = rank, world
        self.next = 0
        self.queue = deque()
        self.running = []
        self.gen = {r: 0 for r in self.req_ids}
        self.finished = 0
        for r in self.req_ids:
            if -(-(self.l_in[r] + self.l_out[r]) // page_size) > cap_pages:
                raise RuntimeError(f"request {r} cannot fit the cap alone")

    def release_arrivals(self, clock):
        while self.next < len(self.req_ids) and self.arrival[self.next] <= clock:
            self.queue.append(self.req_ids[self.next])
            self.next += 1

    def idle(self):
        return not self.running and not self.queue and not self.prefilling

    def done(self):
        return self.idle() and self.next >= len(self.req_ids)

    def next_arrival(self):
        return self.arrival[self.next] if self.next < len(self.req_ids) else None

    def admit_and_grow(self, b_share):
        admitted = preempted = swap_out = swap_in = 0
        while self.queue and len(self.running) < b_share:           # step 2
            r = self.queue[0]
            T = self.l_in[r] + self.gen[r]
            if self.kv.alloc.free < -(-(T + 1) // self.P):
                break
            self.queue.popleft()
            if r in self.swapped:                                      # step 2'
                self.swap_used -= self.swapped.pop(r)
                swap_in += 1
            self.kv.begin(r)
            self.kv.append([r], [T])
            self.running.append(r)
            admitted += 1
        while True:                                                    # step 3
            need = sum(1 for r in self.running if self.kv.ctx[r] % self.P == 0)
            if need <= self.kv.alloc.free:
                break
            victim = self.running.pop()
            held = len(self.kv.pages[victim])
            if self.swap_cap and held <= self.swap_cap - self.swap_used:   # step 3'
                self.swapped[victim] = held
                self.swap_used += held
                swap_out += 1
            self.kv.release(victim)
            self.queue.appendleft(victim)
            preempted += 1
        self.last_swaps = (swap_out, swap_in)
        self.kv.append(self.running, [1] * len(self.running))
        for r in self.running:
            self.gen[r] += 1
        return admitted, preempted

    def step_pd(self, b_share):
        """PD-fusion steps a-c (module docstring).  Returns (admitted, preempted, chunks)."""
        P = self.P
        pre = 0
        while True:                                                    # a
            need = sum(1 for r in self.running if self.kv.ctx[r] % P == 0)
            if need <= self.kv.alloc.free:
                break
            victim = self.prefilling.pop()[0] if self.prefilling else self.running.pop()
            self.kv.release(victim)
            self.queue.appendleft(victim)
            pre += 1
        self.kv.append(self.running, [1] * len(self.running))
        for r in self.running:
            self.gen[r] += 1
        tokens = self.pd_token_budget if self.pd_token_budget > 0 else b_share
        rows = tokens if self.max_rows is None else min(tokens, self.max_rows)
        budget = max(0, rows - len(self.running))                     # b
        chunks, adm, i = [], 0, 0
        while budget > 0:                                              # c
            if i < len(self.prefilling):
                r, done = self.prefilling[i]
                T = self.l_in[r] + self.gen[r]
                k = min(T - done, budget)
                room = (-(-done // P) + self.kv.alloc.free) * P - done
                cut = room < k
                k = min(k, room)
                if k <= 0:
                    break
            elif self.queue and len(self.running) + len(self.prefilling) < b_share:
                r, done = self.queue[0], 0
                T = self.l_in[r] + self.gen[r]
                if self.kv.alloc.free < -(-(T + 1) // P):
                    break
                self.queue.popleft()
                self.kv.begin(r)
                self.prefilling.append([r, 0])
                adm += 1
                k, cut = min(T, budget), False
            else:
                break
            self.kv.append([r], [k])
            self.prefilling[i][1] += k
            chunks.append((r, done, k))
            budget -= k
            i += 1
            if cut:
                break
        self.last_chunks = chunks
        return adm, pre, chunks

    def finish_prefills(self):
        """PD step e: completed prompts join the running batch (admission order)."""
        while self.prefilling and self.prefilling[0][1] == self.l_in[self.prefilling[0][0]] + \
                self.gen[self.prefilling[0][0]]:
            self.running.append(self.prefilling.pop(0)[0])

    def batch(self):
        """The decode launch's batch: (req_ids, ctx, l_in, l_out, pages) in batch order."""
        rs = list(self.running)
        return (rs, [self.kv.ctx[r] for r in rs], [self.l_in[r] for r in rs],
                [self.l_out[r] for r in rs], [list(self.kv.pages[r]) for r in rs])

    def local_stats(self):
        rs, ctx, li, lo, pages = self.batch()
        return ostats.batch_stats(ctx, li, lo, pages, self.P, self.cap)

    def table_hash(self):
        h = FNV_OFFSET
        for r in self.running:
            h = fnv1a64([r, self.kv.ctx[r], len(self.kv.pages[r])] + self.kv.pages[r], h)
        return h

    def retire(self):
        keep, fin = [], 0
        for r in self.running:
            if self.gen[r] == self.l_out[r]:
                self.kv.release(r)
                fin += 1
            else:
                keep.append(r)
        self.running = keep
        self.finished += fin
        return fin


def b_share(b, rank, world, t=0):
    """This rank's share of the global b_t at step t (DP request shards, reading R21): an
    equal split, the b_t mod G remainder going to the ranks r with (r - t) mod G < b_t mod G,
    so the extra slot rotates and a rank whose floor share is 0 (b_t < G) still gets a turn."""
    return b // world + (1 if (rank - t) % world < b % world else 0)


class Replay:
    """Lock-step replay of G rank engines sharing one scheduling decision per step."""

    def __init__(self, ranks, sched_cfg, mem_cap_bytes_total):
        self.ranks = ranks
        self.sched = Scheduler(sched_cfg)
        self.mem_cap = int(mem_cap_bytes_total)
        self.clock = 0
        self.t = 0
        self.b = self.sched.b

    def done(self):
        return all(e.done() for e in self.ranks)

    def step(self, step_ns):
        """One iteration; step_ns = the logged device time (max over ranks).  Returns the record."""
        G = len(self.ranks)
        for e in self.ranks:
            e.release_arrivals(self.clock)
        if all(e.idle() for e in self.ranks):
            nxt = [a for a in (e.next_arrival() for e in self.ranks) if a is not None]
            if not nxt:
                raise RuntimeError("replay finished")
            self.clock = max(self.clock, min(nxt))
            for e in self.ranks:
                e.release_arrivals(self.clock)
        clock0 = self.clock
        adm = pre = n_prefill = 0
        chunks = []
        for e in self.ranks:
            if e.pd:
                a, p, ch = e.step_pd(b_share(self.b, e.rank, G, self.t))
                n_prefill += sum(k for _, _, k in ch)
                chunks.append(ch)
            else:
                a, p = e.admit_and_grow(b_share(self.b, e.rank, G, self.t))
            adm += a
            pre += p
        recs = [e.local_stats() for e in self.ranks]
        batches = [e.batch() for e in self.ranks]
        hashes = [e.table_hash() for e in self.ranks]
        used = [e.kv.alloc.used for e in self.ranks]
        fin = sum(e.retire() for e in self.ranks)
        self.clock += int(step_ns)
        for e in self.ranks:
            e.release_arrivals(self.clock)
        waiting = sum(len(e.queue) + len(e.prefilling) for e in self.ranks)
        for e in self.ranks:
            if e.pd:
                e.finish_prefills()
        for r in recs:
            r["step_ns"] = int(step_ns)
            r["n_waiting"] = 0
        g = ostats.reduce_records(recs, "dp") if G > 1 else dict(recs[0])
        g["n_waiting"] = waiting
        assert g["n_finished"] == fin
        b_t = self.b
        self.b, rationale = self.sched.decide(g, self.mem_cap, waiting)
        rec = dict(t=self.t, clock_ns=clock0, b_t=b_t, n_admitted=adm, n_preempted=pre,
                   n_decode=g["n_active"], n_finished=fin, sum_ctx=g["sum_ctx"],
                   used_pages=sum(used), step_ns=int(step_ns), b_next=self.b, rationale=rationale,
                   L0=self.sched.L0, b_quad=self.sched.bq, b_mem=self.sched.b_mem,
                   b_sla=self.sched.b_sla, table_hash=hashes[0] if G == 1 else tuple(hashes),
                   stats=g, local_stats=recs, batches=batches, n_prefill=n_prefill, chunks=chunks,
                   n_swap_out=sum(e.last_swaps[0] for e in self.ranks),
                   n_swap_in=sum(e.last_swaps[1] for e in self.ranks))
        if any(e.pd for e in self.ranks):
            rec["used_pages"] = g["sum_pages"]   # decode batch pages (prefilling pages excluded)
        self.t += 1
        return rec
