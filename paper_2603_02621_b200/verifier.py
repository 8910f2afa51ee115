"""High-level handle over one libgb context: workspace as a torch tensor, the
torch current stream, result vectors as device tensors.  Marshalling only."""
from __future__ import annotations

import torch

from . import gb


class Verifier:
    """One gb_ctx on one device.

    hi_max : exclusive upper bound of every range this verifier will see
    p_max  : largest fast-path prime bound (default 65521, the largest prime < 2^16)
    origin : even n origin of the MAX_KEY encoding ((n - origin)/2 < 2^40)
    """

    def __init__(self, hi_max: int, p_max: int = 65521, origin: int = 0, device=None, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("libgb needs a CUDA device; there is no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.hi_max, self.p_max, self.origin = hi_max, p_max, origin
        nbytes = gb.gb_ctx_workspace_bytes(hi_max, p_max)
        if nbytes == 0:
            raise ValueError(f"invalid hi_max={hi_max} / p_max={p_max}")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.ctx = gb.gb_ctx_create(self.device.index, origin, hi_max, p_max, self.workspace, self.stream)
        self.n_base, self.R = gb.gb_ctx_info(self.ctx)

    # -- result vectors --------------------------------------------------------
    def new_result(self) -> torch.Tensor:
        r = torch.empty(gb.RESULT_WORDS, dtype=torch.int64, device=self.device)
        gb.gb_result_init(r, self.stream)
        return r

    def finalize(self, result: torch.Tensor) -> None:
        gb.gb_result_finalize(result, self.stream)

    def decode(self, result: torch.Tensor) -> dict:
        return gb.decode_result(result.cpu(), self.origin)

    # -- operations --------------------------------------------------------------
    def verify(self, lo: int, hi: int, result: torch.Tensor, p_max: int | None = None,
               dump: torch.Tensor | None = None, cap: int | None = None, mode: str = "bulk") -> None:
        """mode "bulk": the product path (inverted bulk marking); "pern": the paper's
        per-n gpu3 kernel (NEXT-1 comparison mode)."""
        p = self.p_max if p_max is None else p_max
        if mode == "pern":
            if cap is not None:
                raise ValueError("the per-n mode has no fallback cap hook")
            gb.gb_verify_range_pern(self.ctx, lo, hi, p, result, dump, self.stream)
        elif cap is None:
            gb.gb_verify_range(self.ctx, lo, hi, p, result, dump, self.stream)
        else:
            gb.gb_verify_range_ex(self.ctx, lo, hi, p, cap, result, dump, self.stream)

    def run(self, lo: int, hi: int, p_max: int | None = None, dump: bool = False,
            cap: int | None = None, mode: str = "bulk"):
        """init + verify + finalize; returns (decoded dict, dump tensor or None)."""
        r = self.new_result()
        d = None
        if dump:
            e = 4 if lo < 4 else lo + (lo & 1)
            d = torch.zeros(max(0, (hi - e + 1) // 2), dtype=torch.int32, device=self.device)
        self.verify(lo, hi, r, p_max=p_max, dump=d if (d is not None and d.numel()) else None, cap=cap, mode=mode)
        self.finalize(r)
        self.stream.synchronize()
        return self.decode(r), d

    def run_resident(self, lo: int, hi: int, bits: torch.Tensor, p_max: int | None = None, dump: bool = False):
        """NEXT-2: gpu2-style verification against a resident odd bitset `bits`
        (int64 words [0, n) of the global layout, e.g. sieve_segment(0, n))."""
        r = self.new_result()
        d = None
        if dump:
            e = 4 if lo < 4 else lo + (lo & 1)
            d = torch.zeros(max(0, (hi - e + 1) // 2), dtype=torch.int32, device=self.device)
        gb.gb_verify_range_resident(self.ctx, lo, hi, self.p_max if p_max is None else p_max, bits, bits.numel(), r,
                                    d if (d is not None and d.numel()) else None, self.stream)
        self.finalize(r)
        self.stream.synchronize()
        return self.decode(r), d

    def single_check(self, n: int, p_limit: int = (1 << 64) - 1) -> int:
        """NEXT-3: minimal p <= p_limit with n - p prime for one even n (0 if none)."""
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        gb.gb_single_check(self.ctx, n, p_limit, out, self.stream)
        self.stream.synchronize()
        return int(out.cpu()[0]) & ((1 << 64) - 1)

    def partition_counts(self, lo: int, hi: int, bits: torch.Tensor | None = None) -> torch.Tensor:
        """NEXT-4: c(n) for every even n in [lo_e, hi) (int64 tensor indexed (n - lo_e)/2).
        bits: the odd bitset words [0, n) covering every odd q < hi (sieved here,
        gb_sieve_segment, when not given; needs hi_max >= hi)."""
        if bits is None:
            bits = self.sieve_segment(0, (hi - 3 + 127) // 128)
        e = 4 if lo < 4 else lo + (lo & 1)
        out = torch.empty(max(0, (hi - e + 1) // 2), dtype=torch.int64, device=self.device)
        gb.gb_partition_counts(self.ctx, lo, hi, bits, bits.numel(), out if out.numel() else None, self.stream)
        return out

    def sieve_segment(self, word_lo: int, n_words: int) -> torch.Tensor:
        out = torch.empty(n_words, dtype=torch.int64, device=self.device)
        gb.gb_sieve_segment(self.ctx, word_lo, n_words, out, self.stream)
        return out

    def is_prime(self, x: torch.Tensor) -> torch.Tensor:
        x = x.to(device=self.device, dtype=torch.int64).contiguous()
        out = torch.empty(x.numel(), dtype=torch.uint8, device=self.device)
        gb.gb_is_prime_u64(x, out, x.numel(), self.stream)
        return out

    def close(self) -> None:
        if getattr(self, "ctx", None):
            gb.gb_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
