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
        ctx.import_panel(buf.data_ptr(), n_kept, n_pheno, gidx, n_src)
    return int(buf.numel())


# ----------------------------------------------------------------------------- merging shard outputs
def shard_path(out_path: Path, rank: int) -> Path:
    return Path(f"{out_path}.rank{rank}")


def merge_tsv(shards: list[Path], out_path: Path) -> int:
    """Concatenate THRESHOLD shard TSVs (header once) in rank order; returns records."""
    n = 0
    with open(out_path, "w") as out:
        out.write("\t".join(output.TSV_COLUMNS) + "\n")
        for p in shards:
            with open(p) as fh:
                header = fh.readline()
                if header.rstrip("\n").split("\t") != list(output.TSV_COLUMNS):
                    raise PanelGwasError(f"{p}: not a panelgwas TSV shard")
                for line in fh:
                    out.write(line)
                    n += 1
    return n


def merge_topk(shards: list[Path], out_path: Path, top_k: int, phenotype_names: list[str],
               source_index_of: dict[str, int]) -> int:
    """Per phenotype keep the k best of all shard records by (p, marker source index)."""
    recs = []
    for p in shards:
        recs.extend(output.load_association_records(p))
    lines_of = {}
    for p in shards:
        with open(p) as fh:
            fh.readline()
            for line in fh:
                f = line.rstrip("\n").split("\t")
                lines_of[(f[1], f[12])] = line
    col = {name: j for j, name in enumerate(phenotype_names)}
    recs.sort(key=lambda r: (col[r.phenotype], r.p, source_index_of[r.id]))
    n = 0
    taken: dict[str, int] = {}
    with open(out_path, "w") as out:
        out.write("\t".join(output.TSV_COLUMNS) + "\n")
        for r in recs:
            if taken.get(r.phenotype, 0) >= top_k:
                continue
            taken[r.phenotype] = taken.get(r.phenotype, 0) + 1
            out.write(lines_of[(r.id, r.phenotype)])
            n += 1
    return n


def merge_full(shards: list[Path], out_path: Path) -> int:
    """Concatenate FULL shard matrices (rank order) and their marker sidecars; patch the row count."""
    header = struct.Struct("<16sIQQI")
    rows = 0
    with open(out_path, "wb") as out:
        first = True
        for p in shards:
            blob = Path(p).read_bytes()
            magic, version, m, n_p, code = header.unpack_from(blob)
            if first:
                out.write(header.pack(magic, version, 0, n_p, code))
                first = False
            out.write(blob[header.size:])
            rows += m
        out.seek(len(output.FULL_MAGIC) + 4)
        out.write(struct.pack("<Q", rows))
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
    src = open_genotype_source(config.source)
    try:
        n_markers = src.n_markers
    finally:
        src.close()
    start, stop = shard_span(n_markers, world, rank)
    shard_cfg = replace(config, out_path=shard_path(Path(config.out_path), rank), device=local,
                        summary_to_stderr=False)
    dev = torch.device("cuda", local)

    def panel_hook(ctx, prep):
        # rank 0 prepares + quantizes the panel on its GPU; the zero-variance flags and
        # the quantized limbs reach the other GPUs in two broadcasts (NCCL)
        from .engine import stage_panel

        err = None
        if rank == 0:
            try:
                stage_panel(ctx, prep, n_src)
            except Exception as exc:  # tell the other ranks before re-raising
                err = exc
        flags = [(prep.zero_variance, None if err is None else f"{type(err).__name__}: {err}") if rank == 0 else None]
        dist.broadcast_object_list(flags, 0)
        if err is not None:
            raise err
        if flags[0][1] is not None:
            raise PanelGwasError(f"rank 0 panel preparation failed: {flags[0][1]}")
        if rank != 0:
            prep.set_flags(flags[0][0])
        broadcast_panel(ctx, torch, dist, rank, prep.align.n_kept, len(prep.pheno_names),
                        prep.align.genotype_row_index, n_src, dev)

    src = open_genotype_source(config.source)
    n_src = src.n_samples
    src.close()
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
        dist.broadcast_object_list(box, 0)
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
    dist.all_gather_object(gathered, (summary.to_dict(), summary.phenotype_names) if summary else None)
    names_of = next((g[1] for g in gathered if g is not None), [])
    gathered = [g[0] if g is not None else None for g in gathered]
    result = None
    if rank == 0:
        shards = [shard_path(Path(config.out_path), r) for r in range(world) if gathered[r] is not None]
        first = next(g for g in gathered if g is not None)
        if config.output_mode is engine.OutputMode.FULL:
            records = merge_full(shards, Path(config.out_path)) * first["phenotypes_scanned"]
        elif config.output_mode is engine.OutputMode.TOPK:
            with open(shards[0]) as fh:
                fh.readline()
            src = open_genotype_source(config.source)
            try:
                index = {m.id: m.source_index for m in src.marker_catalog}
            finally:
                src.close()
            records = merge_topk(shards, Path(config.out_path), config.top_k, names_of, index)
        else:
            records = merge_tsv(shards, Path(config.out_path))
        total = dict(first)
        for key in ("markers_scanned", "markers_skipped_monomorphic", "markers_skipped_all_missing", "clamp_count",
                    "p_underflow_count"):
            total[key] = sum(g[key] for g in gathered if g is not None)
        total["n_markers"] = n_markers
        total["records_emitted"] = records
        if config.min_p_sidecar:
            merge_min_p([Path(str(p) + ".minp.tsv") for p in shards], Path(str(config.out_path) + ".minp.tsv"))
        for key in ("time_decode_s", "time_prepare_s", "time_correlate_s", "time_emit_s", "wall_s"):
            total[key] = max(g[key] for g in gathered if g is not None)
        import json

        with open(Path(str(config.out_path) + ".summary.json"), "w") as fh:
            json.dump(total, fh, indent=2, sort_keys=True)
            fh.write("\n")
        for p in [shard_path(Path(config.out_path), r) for r in range(world)]:
            for suffix in ("", ".summary.json", ".markers.tsv", ".phenotypes.txt", ".qc.tsv", ".minp.tsv"):
                q = Path(str(p) + suffix)
                if q.exists():
                    q.unlink()
        result = total
    dist.barrier()
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
