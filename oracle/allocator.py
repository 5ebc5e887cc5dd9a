"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

O2: the KV page allocator.

The paper gives no allocator; it states only that the memory rule "can be
implemented using blocks rather than relying on the number of tokens"
(§III-A after Alg. 1) and that the KV cache is bounded by the
memory left after weights and activations, M_max (§II-B).
Readings (R7-R9):
* pages 0 .. cap_pages-1; an allocation takes the LOWEST-numbered free page,
  so block tables do not depend on the order in which pages were freed;
* within one call, requests are served in the order given (batch order);
* an append is all-or-nothing: if the batch needs more pages than are free,
  nothing changes and the call reports ECAP;
* release returns all of a request's pages.
pages(i) = ceil(ctx_i / P) at every call boundary.
"""
from __future__ import annotations

import heapq


class CapExceeded(Exception):
    """All-or-nothing append would exceed cap_pages; state unchanged."""


class PageAllocator:
    def __init__(self, cap_pages: int):
        if cap_pages < 1:
            raise ValueError("cap_pages must be >= 1")
        self.cap = int(cap_pages)
        self._free = list(range(self.cap))  # a sorted list is a valid min-heap
        self._is_free = [True] * self.cap

    @property
    def free(self) -> int:
        return len(self._free)

    @property
    def used(self) -> int:
        return self.cap - len(self._free)

    def take(self, k: int) -> list[int]:
        """k lowest-numbered free pages, ascending.  Raises CapExceeded (no change)."""
        if k > len(self._free):
            raise CapExceeded(k)
        out = [heapq.heappop(self._free) for _ in range(k)]
        for p in out:
            self._is_free[p] = False
        return out

    def give_back(self, pages) -> None:
        for p in pages:
            if self._is_free[p]:
                raise ValueError(f"double free of page {p}")
            self._is_free[p] = True
            heapq.heappush(self._free, p)


class PagedKV:
    """Request table + allocator: tokens and pages per request (host bookkeeping)."""

    def __init__(self, cap_pages: int, page_size: int):
        self.alloc = PageAllocator(cap_pages)
        self.P = int(page_size)
        self.ctx: dict[int, int] = {}
        self.pages: dict[int, list[int]] = {}

    def begin(self, req: int) -> None:
        if req in self.ctx:
            raise ValueError(f"request {req} already active")
        self.ctx[req] = 0
        self.pages[req] = []

    def pages_needed(self, req: int, n_tok: int) -> int:
        c = self.ctx[req]
        return -(-(c + n_tok) // self.P) - len(self.pages[req])

    def append(self, reqs, n_toks) -> None:
        """All-or-nothing append of n_toks[i] tokens to reqs[i], pages in batch order."""
        need = [self.pages_needed(r, t) for r, t in zip(reqs, n_toks)]
        if sum(need) > self.alloc.free:
            raise CapExceeded(sum(need))
        for r, t, k in zip(reqs, n_toks, need):
            self.pages[r].extend(self.alloc.take(k))
            self.ctx[r] += t

    def release(self, req: int) -> list[int]:
        pg = self.pages.pop(req)
        del self.ctx[req]
        self.alloc.give_back(pg)
        return pg
