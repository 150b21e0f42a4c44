"""CPU ORACLE for NEXT-2, the paged embedding buffer -- TEST INFRASTRUCTURE.

Only ``tests/`` (and ``bench.py``'s reference legs) may import this module;
the product (``libfc``: ``fc_pages_*``, ``fc_paged_copy``) never does, and the
two share no code.

It follows PAPER.md §4.2 "Embedding Buffer Management" (Fig. 10)
and SPEC.md's embed_buffer module step by step, written for
reading rather than speed:

* ``PagedBuffer`` -- the page table.  A request's token s lives in
  slot s mod P of the request's (s div P)-th page, the pages being appended in
  allocation order ("classic virtual-memory paging").  alloc_pages
   appends the minimal number of pages, lowest free ids first, or
  raises OutOfPages with nothing allocated.  ``index`` builds the four indices
  of one iteration (reading R21 in DESIGN.md).  After a read, every
  page whose last token has been read is consumed, and ``free_consumed``
  returns consumed pages to the free list (Fig. 10: "processed blocks
  (e.g., 8 and 11) are promptly freed", a straddling page is freed by
  the read that consumes its last token).
* ``read_chunk`` / ``write_chunk`` -- the data movement, in the paper's four
  steps: the token count and chunk-local position from pv_indptr, the
  page ids from pv_page_indices / pv_page_indptr, the start offset n from
  pv_cu_page_len, then token by token from the n-th token of those pages.

Pinned (tests/test_paged.py, ``-m "not gpu"``): SPEC's worked examples
(S:241-243), a reconstruction of Fig. 10's scenario
(tests/golden/fig10_pages.txt), and randomized operation sequences checked
against flat per-request linear buffers with the table invariants
(S:224).
"""
from __future__ import annotations

import numpy as np


class OutOfPages(Exception):
    """the free list cannot cover an allocation (nothing is allocated)."""


class PageError(Exception):
    """CapacityError / UnwrittenRange / UseAfterFree."""


class PagedBuffer:
    def __init__(self, total_pages: int, page_size: int):
        self.total_pages = total_pages
        self.P = page_size
        self.free = list(range(total_pages))  # kept sorted: lowest id first
        self.pages: dict[int, list[int]] = {}  # request -> every page it was given, in token order
        self.reserved: dict[int, int] = {}
        self.written: dict[int, int] = {}
        self.read: dict[int, int] = {}
        self.consumed_pages: dict[int, set[int]] = {}  # request -> its page positions already consumed
        self.consumed: list[int] = []  # page ids awaiting free_consumed, in order

    # S:237-243 alloc_pages
    def alloc(self, req: int, tokens: int) -> list[int]:
        have = self.pages.get(req, [])
        target = max(self.reserved.get(req, 0), self.written.get(req, 0)) + tokens
        need = -(-target // self.P) - len(have)
        need = max(need, 0)
        if need > len(self.free):
            raise OutOfPages(f"request {req} needs {need} pages, {len(self.free)} free")
        new = self.free[:need]
        self.free = self.free[need:]
        self.pages[req] = have + new
        self.reserved[req] = target
        self.written.setdefault(req, 0)
        self.read.setdefault(req, 0)
        self.consumed_pages.setdefault(req, set())
        return new

    def _page_of(self, req: int, s: int) -> int:
        """Page id holding the request's token s (linear index -> (page, offset))."""
        g = s // self.P
        if g in self.consumed_pages[req]:
            raise PageError(f"UseAfterFree: request {req} token {s} is on a freed page")
        return self.pages[req][g]

    # the four indices of one iteration
    def index(self, op: str, reqs: list[int], counts: list[int]):
        assert op in ("write", "read")
        if len(set(reqs)) != len(reqs):
            raise PageError("a request appears twice in one index")
        for r, c in zip(reqs, counts):  # validate all before changing anything
            if c < 0:
                raise PageError("negative count")
            if c == 0:
                continue
            if r not in self.pages:
                raise PageError(f"request {r} has no pages")
            if op == "write" and self.written[r] + c > len(self.pages[r]) * self.P:
                raise PageError("CapacityError")
            if op == "read" and self.read[r] + c > self.written[r]:
                raise PageError("UnwrittenRange")
        indptr, page_indptr, page_indices, cu_len = [0], [0], [], []
        for r, c in zip(reqs, counts):
            cu = (self.written if op == "write" else self.read).get(r, 0)
            cu_len.append(cu)
            if c > 0:
                first, last = cu // self.P, (cu + c - 1) // self.P
                for g in range(first, last + 1):
                    page_indices.append(self._page_of(r, g * self.P))
                if op == "write":
                    self.written[r] = cu + c
                else:
                    self.read[r] = cu + c
                    # pages whose last token has now been read are consumed
                    for g in range(len(self.pages[r])):
                        if (g + 1) * self.P <= self.read[r] and g not in self.consumed_pages[r]:
                            self.consumed_pages[r].add(g)
                            self.consumed.append(self.pages[r][g])
            indptr.append(indptr[-1] + c)
            page_indptr.append(len(page_indices))
        return indptr, page_indptr, page_indices, cu_len

    # P:494 eager free after the iteration
    def free_consumed(self) -> list[int]:
        out = self.consumed
        self.consumed = []
        self.free = sorted(self.free + out)
        return out

    def release(self, req: int) -> None:
        if req not in self.pages:
            raise PageError(f"unknown request {req}")
        for g, pid in enumerate(self.pages[req]):
            if g not in self.consumed_pages[req]:
                self.consumed.append(pid)
        for d in (self.pages, self.reserved, self.written, self.read, self.consumed_pages):
            del d[req]

    def owned(self) -> int:
        return sum(len(p) - len(self.consumed_pages[r]) for r, p in self.pages.items())


def _token_rows(index, page_size: int):
    """The paper's four steps for every request of the iteration:
    yields (chunk row, page id, slot in page)."""
    indptr, page_indptr, page_indices, cu_len = index
    for i in range(len(cu_len)):
        count = indptr[i + 1] - indptr[i]            # 1. tokens and chunk-local position (pv_indptr)
        pages = page_indices[page_indptr[i]:page_indptr[i + 1]]  # 2. page ids
        n = cu_len[i] % page_size                    # 3. start offset n from pv_cu_page_len
        for k in range(count):                       # 4. tokens from the n-th token of those pages
            s = n + k
            yield indptr[i] + k, pages[s // page_size], s % page_size


def read_chunk(pool: np.ndarray, index, page_size: int) -> np.ndarray:
    """pool [pages, P, cols] -> chunk [pv_indptr[-1], cols]."""
    chunk = np.zeros((index[0][-1],) + pool.shape[2:], dtype=pool.dtype)
    for row, page, slot in _token_rows(index, page_size):
        chunk[row] = pool[page, slot]
    return chunk


def write_chunk(pool: np.ndarray, index, page_size: int, chunk: np.ndarray) -> np.ndarray:
    """A copy of pool with the chunk's rows written into their pages."""
    out = pool.copy()
    for row, page, slot in _token_rows(index, page_size):
        out[page, slot] = chunk[row]
    return out
