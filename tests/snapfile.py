"""Reader of the reference's OSCFSNAP snapshot container (test helper).

Layout as written by io::SnapshotFileWriter (reference
core/src/snapshot.cpp:80-153): magic "OSCFSNAP", u32 version, u32 mode,
u32 ndims, ndims x (8-byte name, u64 length), 4 x 8-byte species names,
u64 config hash, u32 has_spectra [u64 ebins, f64 E0, f64 E1,
4 x (f64 coupling, ebins x f64)], then records {u64 iter, f64 r, f64 dr,
f64 t_wall, payload f64[prod(dims)], u64 fnv1a(payload)}.
"""
from __future__ import annotations

import struct

import numpy as np


def fnv1a(data: bytes) -> int:
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def read(path: str, check_sums: bool = True):
    """Returns (header dict, [(iter, r, dr, t_wall, payload ndarray)])."""
    with open(path, "rb") as f:
        buf = f.read()
    o = 0

    def take(fmt):
        nonlocal o
        v = struct.unpack_from("<" + fmt, buf, o)
        o += struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    if buf[:8] != b"OSCFSNAP":
        raise ValueError(f"{path}: bad magic")
    o = 8
    version, mode, ndims = take("III")
    dims = []
    for _ in range(ndims):
        name = buf[o:o + 8].rstrip(b"\0").decode()
        o += 8
        dims.append((name, take("Q")))
    species = []
    for _ in range(4):
        species.append(buf[o:o + 8].rstrip(b"\0").decode())
        o += 8
    config_hash = take("Q")
    has_spectra = take("I")
    spectra = None
    if has_spectra:
        eb = take("Q")
        E0, E1 = take("dd")
        sp = []
        for _ in range(4):
            c = take("d")
            fvals = np.frombuffer(buf, dtype="<f8", count=eb, offset=o)
            o += 8 * eb
            sp.append((c, fvals.copy()))
        spectra = dict(ebins=eb, E0=E0, E1=E1, species=sp)
    n = 1
    for _, ln in dims:
        n *= ln
    recs = []
    while o < len(buf):
        it = take("Q")
        r, dr, tw = take("ddd")
        raw = buf[o:o + 8 * n]
        if len(raw) != 8 * n:
            raise ValueError(f"{path}: truncated payload")
        payload = np.frombuffer(raw, dtype="<f8").copy()
        o += 8 * n
        cs = take("Q")
        # (byte-serial hash: verified on payloads up to 1 MiB)
        if check_sums and len(raw) <= (1 << 20) and cs != fnv1a(raw):
            raise ValueError(f"{path}: checksum failure")
        recs.append((it, r, dr, tw, payload))
    hdr = dict(version=version, mode=mode, dims=dims, species=species, config_hash=config_hash,
               spectra=spectra)
    return hdr, recs
