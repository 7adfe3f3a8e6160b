"""Multi-GPU scan: contiguous marker shards, one panel broadcast, rank-order merge.

The reference has no distributed mode; SURVEY.md §8e fixes the
B200 decomposition: each marker's statistics depend only on its own row and the
shared panel, so rank g scans the contiguous marker block
[start_g, stop_g) (aligned to 256-marker tiles) with no collective in the scan
loop. The only data-path collective is ONE broadcast of the quantized panel
limbs from rank 0 (pg_ctx_export_panel -> torch.distributed.broadcast ->
pg_ctx_import_panel; NCCL over NVLink for device buffers, gloo for the CPU
tests). Shard outputs concatenate in rank order, which reproduces the
single-GPU (marker, phenotype) record order; TOPK shards merge by
(p, source index). Results are bitwise independent of the GPU count because
every statistic is an exact integer contraction.

Launch: torchrun --nproc-per-node N -m paper_2604_21095_b200.distributed <run flags>
"""

from __future__ import annotations

import os
import struct
from dataclasses import replace
from pathlib import Path

import numpy as np

from . import output
from .errors import PanelGwasError

TILE_MARKERS = 256


def shard_span(n_markers: int, world: int, rank: int, align: int = TILE_MARKERS) -> tuple[int, int]:
    """[start, stop) of rank's contiguous marker block; blocks are `align`-aligned and cover [0, n)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    units = -(-n_markers // align)
    lo = units * rank // world
    hi = units * (rank + 1) // world
    return min(lo * align, n_markers), min(hi * align, n_markers)


def broadcast_bytes(torch, dist, buf, nbytes: int | None, src: int = 0, device=None):
    """Broadcast a byte buffer of unknown size from `src`; returns the buffer on every rank."""
    dev = device if device is not None else "cpu"
    n = torch.tensor([nbytes if nbytes is not None else -1], dtype=torch.int64, device=dev)
    dist.broadcast(n, src)
    if buf is None:
        buf = torch.empty(int(n.item()), dtype=torch.uint8, device=dev)
    dist.broadcast(buf, src)
    return buf


def broadcast_panel(ctx, torch, dist, rank: int, n_kept: int, n_pheno: int, gidx: np.ndarray, n_src: int,
                    device) -> int:
    """Rank 0's resident quantized panel -> every rank's ctx. Returns bytes moved."""
    buf = None
    nbytes = None
    # NCCL moves the device buffer directly; other backends (gloo in the tests) go via host
    wire = device if dist.get_backend() == "nccl" else "cpu"
    if rank == 0:
        nbytes = ctx.panel_bytes()
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        ctx.export_panel(buf.data_ptr())
        if wire == "cpu":
            buf = buf.cpu()
    buf = broadcast_bytes(torch, dist, buf, nbytes, 0, wire)
    if rank != 0:
        if wire == "cpu":
            buf = buf.to(device)
        # the NCCL broadcast (and the copy) complete on torch's stream; the ctx reads the
        # buffer on its own stream, so wait for torch's before handing the pointer over
        torch.cuda.current_stream(device).synchronize()
        ctx.import_panel(buf.data_ptr(), n_kept, n_pheno, gidx, n_src)
    return int(buf.numel())


# ----------------------------------------------------------------------------- merging shard outputs
def shard_path(out_path: Path, rank: int) -> Path:
    return Path(f"{out_path}.rank{rank}")


_COPY_CHUNK = 64 << 20


def _copy_tail(src, out, offset: int, count_lines: bool = False) -> int:
    """Append src[offset:] to the open binary file `out` (kernel-side copy where available);
    returns the number of newlines copied when count_lines."""
    n = 0
    with open(src, "rb") as fh:
        fh.seek(offset)
        if not count_lines and hasattr(os, "sendfile"):
            out.flush()
            size = os.fstat(fh.fileno()).st_size - offset
            while size > 0:
                sent = os.sendfile(out.fileno(), fh.fileno(), None, min(size, 1 << 30))
                if sent <= 0:
                    break
                size -= sent
            if size <= 0:
                return 0
        while True:
            buf = fh.read(_COPY_CHUNK)
            if not buf:
                break
            if count_lines:
                n += buf.count(b"\n")
            out.write(buf)
    return n


def merge_tsv(shards: list[Path], out_path: Path, header: str | None = None) -> int:
    """Concatenate line-oriented shard files (header once) in rank order; returns data lines.

    Used for THRESHOLD record TSVs and their line-aligned .beta.tsv sidecars. The shard
    bodies are copied as bytes in 64 MB chunks (C4's ~1.8e7 null hits are ~2.3 GB of text)."""
    want = header if header is not None else "\t".join(output.TSV_COLUMNS)
    n = 0
    with open(out_path, "wb") as out:
        out.write((want + "\n").encode())
        for p in shards:
            with open(p, "rb") as fh:
                first = fh.readline()
            if first.rstrip(b"\n").decode(errors="replace") != want:
                raise PanelGwasError(f"{p}: not a panelgwas shard of this kind")
            n += _copy_tail(p, out, len(first), count_lines=True)
    return n


def merge_topk(shards: list[Path], out_path: Path, top_k: int, phenotype_names: list[str],
               effect_sizes: bool = False) -> int:
    """Per phenotype keep the k best shard records by (p, marker source index).

    Shard r holds the contiguous marker block [start_r, stop_r) and writes its records in
    (phenotype, p, source index) order, so (phenotype, p, rank, line) orders the union exactly
    as (phenotype, p, source index) would: no lookup by marker ID (IDs may repeat, e.g. '.').
    The optional .beta.tsv sidecars follow the same permutation."""
    col = {name: j for j, name in enumerate(phenotype_names)}
    keys, lines, betas = [], [], []
    for rank, p in enumerate(shards):
        with open(p) as fh:
            if fh.readline().rstrip("\n").split("\t") != list(output.TSV_COLUMNS):
                raise PanelGwasError(f"{p}: not a panelgwas TSV shard")
            shard_lines = fh.readlines()
        if effect_sizes:
            with open(output.beta_sidecar(p)) as fh:
                fh.readline()
                shard_betas = fh.readlines()
            if len(shard_betas) != len(shard_lines):
                raise PanelGwasError(f"{p}: effect-size sidecar is not aligned with the records")
            betas.extend(shard_betas)
        for i, line in enumerate(shard_lines):
            f = line.rstrip("\n").split("\t")
            keys.append((col[f[12]], float(f[11]), rank, i))
        lines.extend(shard_lines)
    order = sorted(range(len(keys)), key=keys.__getitem__)
    taken: dict[int, int] = {}
    chosen = []
    for i in order:
        c = keys[i][0]
        if taken.get(c, 0) < top_k:
            taken[c] = taken.get(c, 0) + 1
            chosen.append(i)
    with open(out_path, "w") as out:
        out.write("\t".join(output.TSV_COLUMNS) + "\n")
        out.writelines(lines[i] for i in chosen)
    if effect_sizes:
        with open(output.beta_sidecar(out_path), "w") as out:
            out.write("\t".join(output.BETA_COLUMNS) + "\n")
            out.writelines(betas[i] for i in chosen)
    return len(chosen)


def merge_qc(shards: list[Path], out_path: Path) -> int:
    """QC sidecars: every shard's skipped-marker rows in rank order, then the phenotype rows
    (identical in every shard: the panel is shared) once, as a single-GPU scan writes them."""
    markers, phenos = [], None
    for p in shards:
        with open(p) as fh:
            header = fh.readline()
            rows = fh.readlines()
        markers.extend(r for r in rows if r.startswith("marker\t"))
        if phenos is None:
            phenos = [r for r in rows if r.startswith("phenotype\t")]
    with open(out_path, "w") as out:
        out.write(header)
        out.writelines(markers)
        out.writelines(phenos or [])
    return len(markers)


def _concat_full_matrices(shards: list[Path], out_path: Path) -> int:
    """Concatenate FULL shard matrices: one header (row count patched), then every shard's
    rows streamed (a C4 shard of 1.1M markers x 20,480 f32 t is ~90 GB)."""
    header = struct.Struct("<16sIQQI")
    rows = 0
    with open(out_path, "wb") as out:
        first = True
        for p in shards:
            with open(p, "rb") as fh:
                magic, version, m, n_p, code = header.unpack(fh.read(header.size))
            if first:
                out.write(header.pack(magic, version, 0, n_p, code))
                first = False
            _copy_tail(p, out, header.size)
            rows += m
        out.flush()
        out.seek(len(output.FULL_MAGIC) + 4)
        out.write(struct.pack("<Q", rows))
    return rows


def merge_full(shards: list[Path], out_path: Path, effect_sizes: bool = False) -> int:
    """Concatenate FULL shard matrices (rank order) and their marker sidecars; patch the row count."""
    rows = _concat_full_matrices(shards, out_path)
    if effect_sizes:
        _concat_full_matrices([output.beta_sidecar(p, full=True) for p in shards],
                              output.beta_sidecar(out_path, full=True))
    side = Path(str(out_path) + ".markers.tsv")
    with open(side, "w") as out:
        out.write("SOURCE_INDEX\tCHR\tID\tPOS\tA1\tA2\tAF\tN_MISS\n")
        for p in shards:
            lines = Path(str(p) + ".markers.tsv").read_text().splitlines(True)[1:]
            out.writelines(lines)
    Path(str(out_path) + ".phenotypes.txt").write_bytes(Path(str(shards[0]) + ".phenotypes.txt").read_bytes())
    return rows


def merge_min_p(shards: list[Path], out_path: Path) -> int:
    """Per phenotype keep the shard row with the largest max |r| (= the smallest p)."""
    best: dict[str, list[str]] = {}
    order: list[str] = []
    for p in shards:
        with open(p) as fh:
            fh.readline()
            for line in fh:
                f = line.rstrip("\n").split("\t")
                if f[0] not in best:
                    order.append(f[0])
                    best[f[0]] = f
                elif float(f[1]) > float(best[f[0]][1]):
                    best[f[0]] = f
    from .engine import MIN_P_COLUMNS

    with open(out_path, "w") as out:
        out.write("\t".join(MIN_P_COLUMNS) + "\n")
        for name in order:
            out.write("\t".join(best[name]) + "\n")
    return len(order)


# ----------------------------------------------------------------------------- the distributed scan
def object_group(dist):
    """Process group for the pickled host collectives (panel metadata, flags, summaries).

    Under NCCL those would be staged through device memory and serialised with the data
    path; a gloo group keeps them on the host so the NCCL communicator carries only the
    one panel broadcast. Returns None (the default group) when the default is already gloo."""
    if dist.get_backend() == "gloo":
        return None
    return dist.new_group(backend="gloo")


def run_scan_distributed(config):
    """torchrun entry: every rank scans its marker shard; rank 0 merges and writes the summary."""
    import torch
    import torch.distributed as dist

    from . import engine
    from .genotypes.types import open_genotype_source

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1:
        return engine.run_scan(config)
    # test hooks: PANELGWAS_DIST_BACKEND=gloo + PANELGWAS_DIST_DEVICE=0 run several ranks on
    # one GPU (host collectives only; no kernel of one rank waits on another)
    backend = os.environ.get("PANELGWAS_DIST_BACKEND", "nccl")
    if os.environ.get("PANELGWAS_DIST_DEVICE"):
        local = int(os.environ["PANELGWAS_DIST_DEVICE"])
        os.environ["PANELGWAS_DEVICE"] = str(local)  # the module-level helper context too
    if not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    objs = object_group(dist)
    src = open_genotype_source(config.source)
    try:
        n_markers = src.n_markers
        n_src = src.n_samples
    finally:
        src.close()
    start, stop = shard_span(n_markers, world, rank)
    shard_cfg = replace(config, out_path=shard_path(Path(config.out_path), rank), device=local,
                        summary_to_stderr=False)
    dev = torch.device("cuda", local)

    def panel_hook(ctx, prep):
        # rank 0 prepares + quantizes the panel on its GPU; the zero-variance flags and the
        # phenotype scales go to the other ranks over the host group, the quantized limbs in
        # the one NCCL broadcast
        from .engine import stage_panel

        err = None
        if rank == 0:
            try:
                stage_panel(ctx, prep, n_src)
            except Exception as exc:  # tell the other ranks before re-raising
                err = exc
        box = [(prep.zero_variance, prep.pheno_sd, None if err is None else f"{type(err).__name__}: {err}")
               if rank == 0 else None]
        dist.broadcast_object_list(box, 0, group=objs)
        if err is not None:
            raise err
        if box[0][2] is not None:
            raise PanelGwasError(f"rank 0 panel preparation failed: {box[0][2]}")
        if rank != 0:
            prep.set_flags(box[0][0])
            prep.pheno_sd = box[0][1]
        broadcast_panel(ctx, torch, dist, rank, prep.align.n_kept, len(prep.pheno_names),
                        prep.align.genotype_row_index, n_src, dev)

    def prep_hook(source):
        # rank 0 parses the phenotype / covariate tables and sends the small metadata; the
        # other ranks never read the (multi-GB) tables
        err = prep = meta = None
        if rank == 0:
            try:
                prep = engine.prepare_panel(config, source)
                meta = engine.panel_metadata(prep)
            except Exception as exc:
                err = exc
        box = [(meta, None if err is None else f"{type(err).__name__}: {err}") if rank == 0 else None]
        dist.broadcast_object_list(box, 0, group=objs)
        if err is not None:
            raise err
        if box[0][1] is not None:
            raise PanelGwasError(f"rank 0 panel preparation failed: {box[0][1]}")
        return prep if rank == 0 else engine.panel_from_metadata(box[0][0])

    # every rank joins the panel broadcast; a rank with an empty shard scans a dummy
    # one-marker range and discards it
    rng = (start, stop) if stop > start else (0, 1)
    summary = engine.run_scan(shard_cfg, marker_range=rng, panel_hook=panel_hook, prep_hook=prep_hook)
    if stop <= start:
        summary = None
    gathered = [None] * world
    dist.all_gather_object(gathered, (summary.to_dict(), summary.phenotype_names) if summary else None, group=objs)
    names_of = next((g[1] for g in gathered if g is not None), [])
    gathered = [g[0] if g is not None else None for g in gathered]
    result = None
    if rank == 0:
        out = Path(config.out_path)
        shards = [shard_path(out, r) for r in range(world) if gathered[r] is not None]
        first = next(g for g in gathered if g is not None)
        beta = config.effect_sizes
        if config.output_mode is engine.OutputMode.FULL:
            records = merge_full(shards, out, effect_sizes=beta) * first["phenotypes_scanned"]
        elif config.output_mode is engine.OutputMode.TOPK:
            records = merge_topk(shards, out, config.top_k, names_of, effect_sizes=beta)
        else:
            records = merge_tsv(shards, out)
            if beta:
                merge_tsv([output.beta_sidecar(p) for p in shards], output.beta_sidecar(out),
                          header="\t".join(output.BETA_COLUMNS))
        total = dict(first)
        for key in ("markers_scanned", "markers_skipped_monomorphic", "markers_skipped_all_missing", "clamp_count",
                    "p_underflow_count"):
            total[key] = sum(g[key] for g in gathered if g is not None)
        total["n_markers"] = n_markers
        total["records_emitted"] = records
        if config.min_p_sidecar:
            merge_min_p([Path(str(p) + ".minp.tsv") for p in shards], Path(str(out) + ".minp.tsv"))
        if config.qc_sidecar:
            merge_qc([Path(str(p) + ".qc.tsv") for p in shards], Path(str(out) + ".qc.tsv"))
        for key in ("time_decode_s", "time_prepare_s", "time_correlate_s", "time_emit_s", "wall_s"):
            total[key] = max(g[key] for g in gathered if g is not None)
        import json

        with open(Path(str(out) + ".summary.json"), "w") as fh:
            json.dump(total, fh, indent=2, sort_keys=True)
            fh.write("\n")
        for p in [shard_path(out, r) for r in range(world)]:
            for suffix in ("", ".summary.json", ".markers.tsv", ".phenotypes.txt", ".qc.tsv", ".minp.tsv",
                           ".beta.tsv", ".beta.bin"):
                q = Path(str(p) + suffix)
                if q.exists():
                    q.unlink()
        result = total
    dist.barrier(group=objs)
    return result


def main(argv=None) -> int:
    from .cli import _scan_config, build_parser

    parser = build_parser()
    args = parser.parse_args(["run", *(argv if argv is not None else __import__("sys").argv[1:])])
    args._parser = parser
    run_scan_distributed(_scan_config(parser, args, args.out))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
