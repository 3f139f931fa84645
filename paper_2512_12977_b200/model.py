"""Toy VLM weights, fingerprint and the B200 device-resident weight layout.

Host side keeps the reference's weight dictionary (fp32 numpy, names and PCG64
draw order of model.py:165-210) so fingerprints and cache staleness checks are
bit-identical to the reference.  `DeviceWeights` is the sm_100a layout the
kernels consume:
  * every projection stored K-major (W^T, [out, in]) in bf16, `out` padded to a
    multiple of 128 (one UMMA M tile), `in` padded to a multiple of 128 (one
    pipeline stage), then PACKED (include/vlcache.h): each 128 x 128 tile is one
    contiguous, pre-swizzled 32 KB block streamed with a single bulk copy;
  * Q and K rows permuted inside each head so the RoPE pair (j, j + hd/2) lands
    in adjacent TMEM lanes (the epilogue exchanges them with one shuffle);
  * gate / up rows interleaved so the SwiGLU pair is adjacent the same way;
  * q, k, v concatenated into one [3*kv, d] projection (one GEMM per layer).
"""
from __future__ import annotations

import hashlib
import json
import struct
from pathlib import Path

import numpy as np

from .config import ModelConfig
from .exceptions import InputError, IntegrityError
from .sequence import Segment, TokenSequence, make_sequence  # noqa: F401  (re-export)

RMS_EPS = 1e-6
WEIGHTS_MAGIC = b"TVLMW001"
BLOCK_NAMES = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "w_gate", "w_up", "w_down")


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# ---------------------------------------------------------------- host weights

def _weight_specs(cfg: ModelConfig):
    """(name, shape, fan_in or None for unscaled, 'ones' flag) in draw order."""
    d, kv, h, pp = cfg.model_dim, cfg.kv_dim, cfg.mlp_hidden, cfg.patch_size ** 2
    block = {"attn_norm": ((d,), "ones"), "wq": ((d, kv), d), "wk": ((d, kv), d), "wv": ((d, kv), d),
             "wo": ((kv, d), kv), "mlp_norm": ((d,), "ones"), "w_gate": ((d, h), d),
             "w_up": ((d, h), d), "w_down": ((h, d), h)}
    yield "embed", (cfg.vocab_size, d), None
    yield "head", (d, cfg.vocab_size), d
    yield "final_norm", (d,), "ones"
    yield "enc_patch_w", (pp, d), pp
    yield "enc_patch_b", (d,), d
    yield "enc_pos", (cfg.tokens_per_image, d), None
    yield "enc_out_norm", (d,), "ones"
    for prefix in ["enc_"] + [f"l{i}_" for i in range(cfg.num_layers)]:
        for name in BLOCK_NAMES:
            shape, fan = block[name]
            yield prefix + name, shape, fan


def init_weights(cfg: ModelConfig) -> dict[str, np.ndarray]:
    rng = np.random.default_rng(np.random.PCG64(cfg.seed))
    out: dict[str, np.ndarray] = {}
    for name, shape, fan in _weight_specs(cfg):
        if fan == "ones":
            out[name] = np.ones(shape, dtype=np.float32)
        elif fan is None:
            out[name] = rng.standard_normal(shape).astype(np.float32)
        else:
            out[name] = (rng.standard_normal(shape) / np.sqrt(fan)).astype(np.float32)
    return out


def _config_json(cfg: ModelConfig) -> str:
    keys = ("num_layers", "num_heads", "model_dim", "kv_dim", "vocab_size", "patch_size",
            "tokens_per_image", "rope_base", "seed")
    return json.dumps({k: getattr(cfg, k) for k in keys}, sort_keys=True)


class ToyVLM:
    """Immutable model: host weights (reference layout) + lazily built device copy."""

    def __init__(self, config: ModelConfig, weights: dict[str, np.ndarray] | None = None):
        self.config = config
        self.w = weights if weights is not None else init_weights(config)
        self._fingerprint: int | None = None
        self._device = None

    @property
    def fingerprint(self) -> int:
        """64-bit id of (config, weights): first 8 bytes of weight_checksum (model.py:221-227)."""
        if self._fingerprint is None:
            self._fingerprint = int.from_bytes(bytes.fromhex(weight_checksum(self))[:8], "big")
        return self._fingerprint

    @property
    def device(self) -> "DeviceWeights":
        if self._device is None:
            self._device = DeviceWeights.from_host(self.config, self.w, self._heads())
        return self._device

    # -- head-parallel attention: one process per GPU, this rank keeps
    # its share of the heads; one all-reduce of the O-projection per layer.
    tp_group = None

    def head_parallel(self, group=None) -> "ToyVLM":
        """Split attention heads over the ranks of `group` (torch.distributed; NCCL on B200)."""
        import torch.distributed as dist
        if self._device is not None:
            raise InputError("head_parallel() must be called before the device weights are built")
        self.tp_group = group if group is not None else dist.group.WORLD
        return self

    def _heads(self):
        if self.tp_group is None:
            return None
        import torch.distributed as dist
        from .sharding import head_split
        return head_split(self.config.num_heads, dist.get_world_size(self.tp_group))[
            dist.get_rank(self.tp_group)]

    @classmethod
    def device_random(cls, config: ModelConfig, seed: int | None = None, tp_group=None,
                      export: dict | None = None) -> "ToyVLM":
        """Random-init weights generated directly on the GPU (benchmarks at 7B shape, where the
        reference's 125 s host init would dominate).  Not bit-identical to init_model.
        export: see DeviceWeights.random (host fp32 copy of the device weights, reference names)."""
        m = cls.__new__(cls)
        m.config = config
        m.w = None
        s = config.seed if seed is None else seed
        m._fingerprint = int.from_bytes(hashlib.sha256(
            (_config_json(config) + f"|device-random|{s}").encode()).digest()[:8], "big")
        if tp_group is not None:
            m.tp_group = tp_group
        m._device = DeviceWeights.random(config, s, m._heads(), export=export)
        return m


def init_model(config: ModelConfig) -> ToyVLM:
    return ToyVLM(config)


def weight_checksum(model: ToyVLM) -> str:
    h = hashlib.sha256(_config_json(model.config).encode())
    for name in sorted(model.w):
        h.update(name.encode())
        h.update(model.w[name].tobytes())
    return h.hexdigest()


def save_weights(model: ToyVLM, path: str | Path) -> None:
    """TVLMW001 blob (model.py:478-490)."""
    names = sorted(model.w)
    header = json.dumps({"config": json.loads(_config_json(model.config)),
                         "tensors": [{"name": n, "shape": list(model.w[n].shape)} for n in names],
                         "dtype": "<f4"}, sort_keys=True).encode()
    with open(path, "wb") as fh:
        fh.write(WEIGHTS_MAGIC + struct.pack("<I", len(header)) + header)
        for n in names:
            fh.write(np.ascontiguousarray(model.w[n], dtype="<f4").tobytes())


def load_model(path: str | Path) -> ToyVLM:
    data = Path(path).read_bytes()
    if data[:8] != WEIGHTS_MAGIC:
        raise IntegrityError(f"{path}: bad magic bytes")
    if len(data) < 12:
        raise IntegrityError(f"{path}: truncated header")
    (hlen,) = struct.unpack("<I", data[8:12])
    try:
        header = json.loads(data[12:12 + hlen])
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise IntegrityError(f"{path}: corrupt header ({exc})") from None
    cfg = ModelConfig(**header["config"])
    w, off = {}, 12 + hlen
    for spec in header["tensors"]:
        nbytes = int(np.prod(spec["shape"])) * 4
        chunk = data[off:off + nbytes]
        if len(chunk) != nbytes:
            raise IntegrityError(f"{path}: truncated tensor {spec['name']}")
        w[spec["name"]] = np.frombuffer(chunk, dtype="<f4").reshape(spec["shape"]).copy()
        off += nbytes
    if off != len(data):
        raise IntegrityError(f"{path}: trailing bytes after tensors")
    return ToyVLM(cfg, w)


# ---------------------------------------------------------------- KV results

class KVTensors:
    """Per-layer pre-RoPE keys/values [L, seq_len, kv_dim].

    Either plain arrays (as in the reference) or device-backed: `keys`/`values`
    then materialise fp32 numpy on first access, `device_keys()`/`device_values()`
    return the bf16 device tensors without a host copy.
    """

    def __init__(self, keys=None, values=None, *, loader=None):
        self._keys, self._values, self._loader = keys, values, loader
        self._dev = None

    def _device(self):
        if self._dev is None:
            self._dev = self._loader()
        return self._dev

    def device_keys(self):
        return self._device()[0]

    def device_values(self):
        return self._device()[1]

    @property
    def keys(self) -> np.ndarray:
        if self._keys is None:
            self._keys = self._device()[0].float().cpu().numpy()
        return self._keys

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._device()[1].float().cpu().numpy()
        return self._values

    @property
    def seq_len(self) -> int:
        return int(self._device()[0].shape[1]) if self._keys is None else self._keys.shape[1]

    def check_finite(self) -> None:
        if not (np.isfinite(self.keys).all() and np.isfinite(self.values).all()):
            raise InputError("non-finite KV entries")


# ---------------------------------------------------------------- device layout

def rope_inv_freq(head_dim: int, base: float) -> np.ndarray:
    """fp32 inverse frequencies exactly as model.py:132."""
    half = head_dim // 2
    return base ** (-np.arange(half, dtype=np.float32) * (2.0 / head_dim))


def rope_tables_np(n_pos: int, head_dim: int, base: float):
    ang = np.arange(n_pos, dtype=np.float32)[:, None] * rope_inv_freq(head_dim, base)
    return np.cos(ang, dtype=np.float32), np.sin(ang, dtype=np.float32)


def rope_row_perm(kv: int, hd: int) -> np.ndarray:
    """Device row r -> original feature: within a head, (2t, 2t+1) <- (t, t + hd/2)."""
    t = np.arange(hd // 2)
    inner = np.stack([t, t + hd // 2], axis=1).reshape(-1)
    return (np.arange(kv // hd)[:, None] * hd + inner[None, :]).reshape(-1)


class DeviceWeights:
    """bf16 K-major weights + fp32 norms + RoPE tables on cuda:0 (see module doc)."""

    def __init__(self, cfg: ModelConfig, heads: tuple[int, int] | None = None):
        """heads = (first head, count) of this rank under head-parallel attention (None = all):
        Q/K/V keep only those heads' output rows, O only their input columns; the MLP, head and
        vision encoder stay whole."""
        import torch
        from . import _native

        if not torch.cuda.is_available():
            raise _native.NativeError("no CUDA device: the B200 path has no CPU fallback")
        _native.load()
        self.cfg = cfg
        self.h0, self.heads = heads if heads is not None else (0, cfg.num_heads)
        self.kv = self.heads * cfg.head_dim                 # local K/V width (this rank's heads)
        self.c0, self.c1 = self.h0 * cfg.head_dim, self.h0 * cfg.head_dim + self.kv
        d, kv, h = cfg.model_dim, self.kv, cfg.mlp_hidden
        self.kd = _round_up(d, 128)         # K of projections fed by d-wide rows
        self.kkv = _round_up(kv, 128)       # K of the O projection
        self.kh = _round_up(h, 128)         # K of the down projection
        self.kp = _round_up(cfg.patch_size ** 2, 128)
        self.n_qkv = _round_up(3 * kv, 128)
        self.n_d = _round_up(d, 128)
        self.n_gu = _round_up(2 * h, 128)
        self.n_vocab = _round_up(cfg.vocab_size, 128)
        self.perm = rope_row_perm(kv, cfg.head_dim)
        self.enc_kv = cfg.kv_dim            # the encoder is never head-split
        self.n_qkv_enc = _round_up(3 * cfg.kv_dim, 128)
        self.kkv_enc = _round_up(cfg.kv_dim, 128)
        self.layers: list[dict] = []
        self.cos = self.sin = self.cs = None
        self.tab_rows = 0

    # -- construction
    @staticmethod
    def _kmajor(torch, w_in_out, n_pad, k_pad, row_index=None):
        """[in, out] fp32 (host or device) -> bf16 [n_pad, k_pad] with W^T rows (optionally reordered)."""
        t = w_in_out if isinstance(w_in_out, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(w_in_out))
        t = t.cuda(non_blocking=True).t()
        if row_index is not None:
            t = t[torch.as_tensor(row_index, device="cuda")]
        out = torch.zeros(n_pad, k_pad, dtype=torch.bfloat16, device="cuda")
        out[:t.shape[0], :t.shape[1]] = t.to(torch.bfloat16)
        return out

    def _block(self, torch, get, whole: bool = False):
        """Device tensors of one transformer block; `get(name)` returns [in, out] fp32.  Unless
        `whole`, attention weights are cut to this rank's heads."""
        cfg = self.cfg
        h = cfg.mlp_hidden
        if whole:
            kv, n_qkv, kkv, perm = cfg.kv_dim, self.n_qkv_enc, self.kkv_enc, rope_row_perm(cfg.kv_dim, cfg.head_dim)
            c0, c1 = 0, cfg.kv_dim
        else:
            kv, n_qkv, kkv, perm, c0, c1 = self.kv, self.n_qkv, self.kkv, self.perm, self.c0, self.c1
        full_get = get
        drawn = {}

        def get(name):                      # noqa: F811 -- head slice of the attention weights
            if name not in drawn:           # one draw per tensor (get() may be asked twice)
                drawn[name] = full_get(name)
            w = drawn[name]
            if name in ("wq", "wk", "wv"):
                return w[:, c0:c1]
            if name == "wo":
                return w[c0:c1, :]
            return w
        wqkv = torch.zeros(n_qkv, self.kd, dtype=torch.bfloat16, device="cuda")
        wqkv[0:kv] = self._kmajor(torch, get("wq"), kv, self.kd, perm)
        wqkv[kv:2 * kv] = self._kmajor(torch, get("wk"), kv, self.kd, perm)
        wqkv[2 * kv:3 * kv] = self._kmajor(torch, get("wv"), kv, self.kd)
        wqkv_plain = torch.zeros_like(wqkv)
        wqkv_plain[0:kv] = self._kmajor(torch, get("wq"), kv, self.kd)
        wqkv_plain[kv:2 * kv] = self._kmajor(torch, get("wk"), kv, self.kd)
        wqkv_plain[2 * kv:3 * kv] = wqkv[2 * kv:3 * kv]
        gu = torch.zeros(self.n_gu, self.kd, dtype=torch.bfloat16, device="cuda")
        g = self._kmajor(torch, get("w_gate"), h, self.kd)
        u = self._kmajor(torch, get("w_up"), h, self.kd)
        gu[0:2 * h:2], gu[1:2 * h:2] = g, u
        def norm(x):
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
            return t.float().cuda().contiguous()
        return {"wqkv": PackedWeight(wqkv), "wqkv_plain": PackedWeight(wqkv_plain),
                "wo": PackedWeight(self._kmajor(torch, get("wo"), self.n_d, kkv)),
                "wgu": PackedWeight(gu), "wd": PackedWeight(self._kmajor(torch, get("w_down"), self.n_d, self.kh)),
                "attn_norm": norm(get("attn_norm")), "mlp_norm": norm(get("mlp_norm"))}

    @classmethod
    def from_host(cls, cfg: ModelConfig, w: dict[str, np.ndarray], heads=None) -> "DeviceWeights":
        import torch
        self = cls(cfg, heads)
        for i in range(cfg.num_layers):
            blk = self._block(torch, lambda n, i=i: w[f"l{i}_{n}"])
            blk.pop("wqkv_plain")
            self.layers.append(blk)
        self.enc = self._block(torch, lambda n: w[f"enc_{n}"], whole=True)
        self.enc["patch_w"] = PackedWeight(self._kmajor(torch, w["enc_patch_w"], self.n_d, self.kp))
        self.enc["patch_b"] = torch.from_numpy(w["enc_patch_b"]).cuda()
        self.enc["pos"] = torch.from_numpy(np.ascontiguousarray(w["enc_pos"])).cuda()
        self.enc["out_norm"] = torch.from_numpy(w["enc_out_norm"]).cuda()
        self.embed = torch.from_numpy(w["embed"]).cuda().to(torch.bfloat16)
        self.final_norm = torch.from_numpy(w["final_norm"]).cuda()
        self.head = PackedWeight(self._kmajor(torch, w["head"], self.n_vocab, self.kd))
        torch.cuda.synchronize()
        return self

    @classmethod
    def random(cls, cfg: ModelConfig, seed: int, heads=None, export: dict | None = None) -> "DeviceWeights":
        """Same distributions as model.py:165-210 (N(0,1)/sqrt(fan_in), unit norms), drawn on device
        (the full tensors are drawn on every rank, so head slices agree across ranks).

        export: if a dict, it receives the weights the device holds as host fp32 arrays in the
        reference's names and [in, out] layout (bf16 values widened), so a CPU reference can run
        on exactly the same model (tests / bench parity at the 7B shape)."""
        import torch
        self = cls(cfg, heads)
        g = torch.Generator(device="cuda").manual_seed(int(seed))
        d, kv, h, pp = cfg.model_dim, cfg.kv_dim, cfg.mlp_hidden, cfg.patch_size ** 2
        shapes = {"wq": (d, kv), "wk": (d, kv), "wv": (d, kv), "wo": (kv, d), "w_gate": (d, h),
                  "w_up": (d, h), "w_down": (h, d)}
        prefix = [""]

        def keep(name, t, rounded=True):
            if export is not None:
                v = t.to(torch.bfloat16).float() if rounded else t.float()
                export[prefix[0] + name] = v.cpu().numpy()
            return t

        def gen(name):
            if name.endswith("norm"):
                return keep(name, torch.ones(d, device="cuda"), rounded=False)
            shape = shapes[name]
            return keep(name, torch.randn(shape, device="cuda", generator=g) / float(np.sqrt(shape[0])))
        for i in range(cfg.num_layers):
            prefix[0] = f"l{i}_"
            blk = self._block(torch, gen)
            blk.pop("wqkv_plain")
            self.layers.append(blk)
        prefix[0] = "enc_"
        self.enc = self._block(torch, gen, whole=True)
        self.enc["patch_w"] = PackedWeight(self._kmajor(
            torch, keep("patch_w", torch.randn(pp, d, device="cuda", generator=g) / float(np.sqrt(pp))),
            self.n_d, self.kp))
        self.enc["patch_b"] = keep("patch_b", torch.randn(d, device="cuda", generator=g) / float(np.sqrt(d)),
                                   rounded=False)
        self.enc["pos"] = keep("pos", torch.randn(cfg.tokens_per_image, d, device="cuda", generator=g),
                               rounded=False)
        self.enc["out_norm"] = keep("out_norm", torch.ones(d, device="cuda"), rounded=False)
        prefix[0] = ""
        self.embed = keep("embed", torch.randn(cfg.vocab_size, d, device="cuda", generator=g).to(torch.bfloat16))
        self.final_norm = keep("final_norm", torch.ones(d, device="cuda"), rounded=False)
        head = torch.zeros(self.n_vocab, self.kd, dtype=torch.bfloat16, device="cuda")
        for r0 in range(0, cfg.vocab_size, 16384):   # chunked to bound the fp32 transient
            r1 = min(cfg.vocab_size, r0 + 16384)
            head[r0:r1, :d] = (torch.randn(r1 - r0, d, device="cuda", generator=g)
                               / float(np.sqrt(d))).to(torch.bfloat16)
        self.head = PackedWeight(head)
        if export is not None:
            export["head"] = np.ascontiguousarray(head[:cfg.vocab_size, :d].float().cpu().numpy().T)
        del head
        torch.cuda.synchronize()
        return self

    # -- RoPE tables (exact reference formula, computed on host)
    def ensure_positions(self, n: int) -> None:
        import torch
        if n <= self.tab_rows:
            return
        rows = max(n, 2 * self.tab_rows, 1024)
        c, s = rope_tables_np(rows, self.cfg.head_dim, self.cfg.rope_base)
        self.cos = torch.from_numpy(c).cuda()
        self.sin = torch.from_numpy(s).cuda()
        # interleaved copy for the QKV epilogue: per row, (cos t, cos t+1, sin t, sin t+1) for even t
        h2 = c.shape[1]
        cs = np.stack([c.reshape(rows, h2 // 2, 2), s.reshape(rows, h2 // 2, 2)], axis=2).reshape(rows, 2 * h2)
        self.cs = torch.from_numpy(np.ascontiguousarray(cs)).cuda()
        self.tab_rows = rows

    def bytes_per_layer(self) -> int:
        l0 = self.layers[0]
        return sum(int(l0[k].t.numel()) * 2 for k in ("wqkv", "wo", "wgu", "wd"))


class PackedWeight:
    """A [n, k] K-major bf16 weight in the packed streaming layout (row tile 128)."""

    def __init__(self, dense):
        from . import _native
        self.n, self.k = int(dense.shape[0]), int(dense.shape[1])
        self.t = _native.pack(dense, 128)

    def data_ptr(self) -> int:
        return self.t.data_ptr()
