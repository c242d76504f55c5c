"""Request data parallelism over the GPUs of one box with a document-sharded KV store.

* One process (and one Engine) per GPU. Every chunk has exactly one OWNER rank, chosen by document
  (owner = FNV-1a(doc id) mod world, so all chunks of a document are co-resident); only the owner
  prefills it into its HBM store.
* Ranks exchange their store directories with one all_gather_object over the process group. A directory
  is the engine's own serialised blob (tkv_store_export_directory: chunk id -> page list, token count,
  framed tokens, plus the pool's CUDA-IPC handle, model fingerprint and page geometry), and every rank
  registers the other ranks' blobs with tkv_store_import_directory, which rejects a peer built under a
  different model or page geometry and any page index outside the peer's pool. The blob format is in
  include/tkv.h, so a C/C++ host shards the same way over its own transport (MPI, NCCL, sockets). No collective runs on the data path: the gather kernel of a
  request reads a remote chunk's pages directly from the owner's HBM over NVLink (P2P loads fused
  with the RoPE re-rotation), or the chunk is copied once into the local store (cache policy).
* The router sends a request to the rank owning most of its chunk tokens, breaking ties by load.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def owner_of(doc_id: str, world: int) -> int:
    """Owner rank of every chunk of document `doc_id` (ChunkRecord.doc_id, retrieval.hpp:25-30)."""
    return fnv1a64(doc_id.encode()) % world if world > 1 else 0


_DIR_HEAD = struct.Struct("<4sIQQqq64sq")


def pack_directory(fingerprint: int, page_bytes: int, page_tokens: int, pool_pages: int, ipc: bytes, entries) -> bytes:
    """The tkv_store_export_directory blob layout (include/tkv.h); entries: (id, length, pages, framed)."""
    out = [_DIR_HEAD.pack(b"TKVD", 1, fingerprint, page_bytes, page_tokens, pool_pages, ipc, len(entries))]
    for cid, length, pages, framed in sorted(entries, key=lambda e: e[0]):
        pages = np.asarray(pages, np.int32)
        framed = np.asarray(framed if framed is not None else [], np.int32)
        out += [struct.pack("<Qqq", cid, length, len(pages)), pages.tobytes(), struct.pack("<q", len(framed)),
                framed.tobytes()]
    return b"".join(out)


def parse_directory(blob: bytes) -> dict:
    """Decode a directory blob (host-side inspection and tests; the engine validates it itself on import)."""
    magic, ver, fp, pb, pt, npages, ipc, n = _DIR_HEAD.unpack_from(blob, 0)
    if magic != b"TKVD" or ver != 1:
        raise ValueError("not a version-1 store directory blob")
    at, entries = _DIR_HEAD.size, []
    for _ in range(n):
        cid, length, np_ = struct.unpack_from("<Qqq", blob, at)
        at += 24
        pages = np.frombuffer(blob, np.int32, np_, at).tolist()
        at += 4 * np_
        (nf,) = struct.unpack_from("<q", blob, at)
        at += 8
        framed = np.frombuffer(blob, np.int32, nf, at).tolist()
        at += 4 * nf
        entries.append((cid, length, pages, framed or None))
    return {"fingerprint": fp, "page_bytes": pb, "page_tokens": pt, "pool_pages": npages, "ipc": ipc,
            "entries": entries}


@dataclass
class DirEntry:
    chunk_id: int
    owner: int
    length: int
    pages: list
    framed: list | None = None


@dataclass
class ShardedStore:
    """Per-rank view of the sharded store. `engine` is a turbokv.Engine (or any object with the same
    ingest_chunks / chunk_pages / export_ipc / attach_ipc / register_remote / fetch_remote methods)."""
    engine: object
    rank: int
    world: int
    directory: dict = field(default_factory=dict)  # chunk id -> DirEntry (all ranks' chunks)
    load: list = field(default_factory=list)

    def __post_init__(self):
        self.load = [0] * self.world

    @staticmethod
    def slot_of(rank: int, peer: int) -> int:
        """Peer slot (1..15) under which `rank` maps `peer`'s page pool."""
        return peer + 1 if peer < rank else peer

    def ingest(self, payloads, doc_ids) -> list:
        """Prefill the chunks this rank owns; returns the content ids of ALL chunks (computed without
        prefilling, since ids depend only on tokens and the model fingerprint)."""
        from . import turbokv as T
        fp = self.engine.fingerprint()
        ids = [T.chunk_content_id(T.frame_chunk(p), fp) for p in payloads]
        mine = [i for i, d in enumerate(doc_ids) if owner_of(d, self.world) == self.rank]
        if mine:
            got = self.engine.ingest_chunks([payloads[i] for i in mine])
            assert got == [ids[i] for i in mine]
        for i in mine:
            pages, length = self.engine.chunk_pages(ids[i])
            self.directory[ids[i]] = DirEntry(ids[i], self.rank, length, pages.tolist(),
                                              T.frame_chunk(payloads[i]).tolist())
        return ids

    def exchange(self, group=None, all_gather_object=None) -> None:
        """Share directory blobs; register every peer's chunks under its slot (validated by the engine)."""
        if self.world == 1:
            return
        import torch.distributed as dist
        gather = all_gather_object or dist.all_gather_object
        local = {"rank": self.rank, "blob": self.engine.export_directory(),
                 "dir": [vars(e) for e in self.directory.values() if e.owner == self.rank]}
        everyone = [None] * self.world
        gather(everyone, local, group=group) if all_gather_object is None else gather(everyone, local)
        for peer in everyone:
            if peer["rank"] == self.rank:
                continue
            slot = self.slot_of(self.rank, peer["rank"])
            self.engine.import_directory(slot, peer["blob"])
            for e in peer["dir"]:
                entry = DirEntry(**e)
                self.directory[entry.chunk_id] = entry

    def route(self, chunk_ids) -> int:
        """Rank for a request: most locally-owned chunk tokens, then least loaded."""
        owned = [0] * self.world
        for cid in chunk_ids:
            e = self.directory.get(cid)
            if e is not None:
                owned[e.owner] += e.length
        best = max(range(self.world), key=lambda r: (owned[r], -self.load[r], -r))
        self.load[best] += 1
        return best

    def remote_fraction(self, chunk_ids) -> float:
        tot = sum(self.directory[c].length for c in chunk_ids)
        rem = sum(self.directory[c].length for c in chunk_ids if self.directory[c].owner != self.rank)
        return rem / tot if tot else 0.0

    def cache_remote(self, chunk_ids) -> None:
        """Fetch-once policy: copy this request's remote chunks into the local store."""
        for cid in chunk_ids:
            e = self.directory[cid]
            if e.owner != self.rank:
                self.engine.fetch_remote(cid)
                self.directory[cid] = DirEntry(cid, self.rank, e.length, [], e.framed)
