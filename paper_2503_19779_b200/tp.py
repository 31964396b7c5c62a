"""Tensor-parallel plumbing: bootstrap the NCCL communicator used by ALLREDUCE_SUM nodes.

torch.distributed (any backend) only carries the 128-byte ncclUniqueId from rank 0 to the others
(P:L857-878 TP setting); the communicator itself is created and owned through the
C ABI (cgx_nccl_comm_init) and the collective is captured inside each rank's graph.
"""
from __future__ import annotations

from . import cgx


def broadcast_unique_id(group=None) -> bytes:
    import torch.distributed as dist
    obj = [cgx.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                               group=group)
    return obj[0]


def nccl_bootstrap(device: int, group=None) -> int:
    """Create this rank's ncclComm_t (returned as an integer handle; destroy with
    cgx.nccl_comm_destroy)."""
    import torch.distributed as dist
    uid = broadcast_unique_id(group)
    return cgx.nccl_comm_init(dist.get_world_size(group), dist.get_rank(group), uid, device)


class PeerRegions:
    """Multi-process setup of the peer-memory all-reduce (cgx_chain_set_peers): every rank owns one
    zero-filled region of cgx_peer_buffer_bytes() in a DEDICATED allocation on its own GPU
    (cgx_device_alloc: the CUDA IPC handle maps a whole allocation, so a sub-allocation of torch's
    caching allocator would land at the wrong offset in the peer), exports its IPC handle, gathers
    every rank's handle through the torch process group and maps the peers' regions into this
    process (cgx_ipc_open; peer access over NVLink). `bases` is then the per-rank pointer list the
    chain takes. Keep the object alive as long as the chain; close() unmaps and frees."""

    def __init__(self, world: int, rank: int, max_elems: int, device, group=None, max_allreduces: int = 64):
        import torch
        import torch.distributed as dist
        dev = torch.device(device)
        self.own = cgx.device_alloc(dev.index if dev.index is not None else torch.cuda.current_device(),
                                    cgx.peer_buffer_bytes(world, max_elems, max_allreduces))
        handle = cgx.ipc_handle(self.own)
        gathered = [None] * world
        dist.all_gather_object(gathered, handle, group=group)
        self.opened, self.bases = [], []
        for r, h in enumerate(gathered):
            if r == rank:
                self.bases.append(self.own)
            else:
                p = cgx.ipc_open(h)
                self.opened.append(p)
                self.bases.append(p)
        self.world, self.rank, self.max_elems, self.max_allreduces = world, rank, max_elems, max_allreduces

    def peers(self) -> tuple:
        return (self.rank, self.world, self.bases, self.max_elems, self.max_allreduces)

    def close(self):
        for p in self.opened:
            cgx.ipc_close(p)
        self.opened = []
        if self.own:
            cgx.device_free(self.own)
            self.own = 0


def share_fd(fd, rank: int, world: int, group=None) -> int:
    """Rank 0's open file descriptor `fd` duplicated into every rank of the process group (same node):
    rank 0 listens on a Unix socket whose path travels through the group, each other rank connects
    and receives the descriptor (SCM_RIGHTS). Returns this rank's descriptor (rank 0: `fd` itself);
    the caller closes it."""
    import os
    import socket
    import tempfile
    import time

    import torch.distributed as dist
    path = None
    if rank == 0:
        path = os.path.join(tempfile.mkdtemp(prefix="cgx_fd_"), "sock")
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path)
        srv.listen(max(1, world - 1))
    meta = [path]
    dist.broadcast_object_list(meta, src=0, group=group)
    path = meta[0]
    if rank == 0:
        for _ in range(world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"fd"], [fd])
            conn.close()
        srv.close()
        os.unlink(path)
        os.rmdir(os.path.dirname(path))
        return fd
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    for _ in range(1200):                       # rank 0 may not be listening yet
        try:
            cli.connect(path)
            break
        except (FileNotFoundError, ConnectionRefusedError):
            time.sleep(0.05)
    _, fds, _, _ = socket.recv_fds(cli, 16, 1)
    cli.close()
    return fds[0]


class MulticastRegion:
    """Multi-process setup of the NVLS all-reduce (cgx_chain_set_multicast): rank 0 creates the
    multicast object for `world` devices and exports it as a POSIX file descriptor, which reaches
    the other ranks over a Unix socket (SCM_RIGHTS; the socket path travels through the torch
    process group); every rank adds its device, waits for the others, binds a zero-filled region of
    cgx_mc_buffer_bytes() and maps it (its own copy + the multicast address). world = 1 needs no
    process group. Keep the object alive as long as the chain; close() releases the region."""

    def __init__(self, world: int, rank: int, max_elems: int, device, group=None, max_allreduces: int = 64):
        import os

        import torch
        dev = torch.device(device)
        self.device = dev.index if dev.index is not None else torch.cuda.current_device()
        if not cgx.mc_supported(self.device):
            raise cgx.CgxError(cgx.E_UNSUPPORTED, "MulticastRegion",
                               "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0 on this device")
        nbytes = cgx.mc_buffer_bytes(max_elems, max_allreduces)
        if world == 1:
            self.handle, self.size = cgx.mc_create(1, nbytes, self.device)
        else:
            import torch.distributed as dist
            err, fd = None, -1
            if rank == 0:
                try:   # (a refusal must reach every rank, or they would wait for the descriptor forever)
                    self.handle, self.size = cgx.mc_create(world, nbytes, self.device)
                    fd = cgx.mc_export_fd(self.handle)
                except cgx.CgxError as exn:
                    err = str(exn)
            meta = [self.size if rank == 0 and err is None else None, err]
            dist.broadcast_object_list(meta, src=0, group=group)
            self.size, err = meta
            if err is not None:
                raise cgx.CgxError(cgx.E_CUDA, "MulticastRegion", f"rank 0: {err}")
            fd = share_fd(fd if rank == 0 else None, rank, world, group)
            if rank != 0:
                self.handle = cgx.mc_import_fd(fd)
            os.close(fd)
        cgx.mc_add_device(self.handle, self.device)
        if world > 1:
            import torch.distributed as dist
            dist.barrier(group=group)                     # every device added before any bind
        self.uc, self.mc = cgx.mc_bind_map(self.handle, self.device, self.size)
        if world > 1:
            import torch.distributed as dist
            dist.barrier(group=group)
        self.world, self.rank, self.max_elems, self.max_allreduces = world, rank, max_elems, max_allreduces

    def multicast(self) -> tuple:
        return (self.world, self.uc, self.mc, self.max_elems, self.max_allreduces)

    def close(self):
        if self.uc:
            cgx.mc_release(self.uc)
            self.uc = 0
