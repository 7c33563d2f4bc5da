"""CPU oracle of the occupancy calculator's block choice (R-24).

TEST INFRASTRUCTURE ONLY: imported by tests/, never by the product package.

The paper asks cudaOccupancyMaxPotentialBlockSize for "the optimal thread block size for a
kernel".  That API maximises the number of resident threads per SM: for each candidate
block size it takes the number of blocks an SM can hold, limited independently by

  * threads:   floor(max_threads_per_sm / (warps_per_block * 32))
  * blocks:    the per-SM block slot limit (32 on compute capability 9.x / 10.0)
  * registers: registers are allocated per warp in units of 256 from four sub-partitions of
               regs_per_sm / 4 each, so warps_per_sm = 4 * floor((regs_per_sm / 4) /
               roundup(regs_per_thread * 32, 256)) and the limit is floor(warps_per_sm /
               warps_per_block)
  * shared memory: floor(smem_per_sm / roundup(static + dynamic + reserved_per_block, 128))

and keeps the best product blocks x threads, scanning block sizes from the largest down, so a
tie goes to the larger block.  This module writes that rule out from the function's attributes
(registers, static shared memory) and the device's limits; the library calls the CUDA API
itself, so the two share nothing but the inputs.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class Device:
    max_threads_per_sm: int = 2048
    max_blocks_per_sm: int = 32
    regs_per_sm: int = 65536
    smem_per_sm: int = 233472          # 228 KiB (B200: the largest carve-out)
    reserved_smem_per_block: int = 1024
    reg_unit: int = 256                # registers per warp are allocated in these units
    sub_partitions: int = 4
    smem_unit: int = 128


def _roundup(x: int, u: int) -> int:
    return -(-x // u) * u


def blocks_per_sm(threads: int, regs_per_thread: int, static_smem: int, dynamic_smem: int,
                  dev: Device = Device()) -> int:
    warps = -(-threads // 32)
    lim = [dev.max_threads_per_sm // (warps * 32), dev.max_blocks_per_sm]
    if regs_per_thread > 0:
        per_warp = _roundup(regs_per_thread * 32, dev.reg_unit)
        warps_sm = dev.sub_partitions * ((dev.regs_per_sm // dev.sub_partitions) // per_warp)
        lim.append(warps_sm // warps)
    smem = static_smem + dynamic_smem + dev.reserved_smem_per_block
    lim.append(dev.smem_per_sm // _roundup(smem, dev.smem_unit))
    return max(0, min(lim))


def choose(candidates, dev: Device = Device()) -> int:
    """Index of the candidate with the most resident warps per SM, ties -> the larger block.
    candidates: list of (threads, regs_per_thread, static_smem, dynamic_smem); threads
    ascending; a candidate with threads == 0 or no implementation passes regs = -1."""
    best, best_w = -1, -1
    for i, (t, r, s, d) in enumerate(candidates):
        if r < 0:
            continue
        w = blocks_per_sm(t, r, s, d, dev) * t // 32
        if w > 0 and w >= best_w:
            best, best_w = i, w
    return best
