"""The configuration kernels and the 2-D driver program as ``.lope`` source text.

Input data for the reference's own frontend and ``Machine`` (``lopec``): used by
``tests/golden/gen_golden.py`` to generate fixtures and by ``bench.py --impl
reference`` to time the reference ``Machine`` on the same program -- test and
benchmark infrastructure only, like the rest of ``oracle/``.  Each kernel is the
stencil SURVEY §8(d) names for a BASELINE configuration; ``MAIN_2D`` is the loop of
``/root/reference/pkg/corpus/laplacian.lope`` (HALO_TRANSFER then a device
``do concurrent`` launch, ``nsteps`` times) around it.
"""

KERNEL_SRC = {
    "heat2d": ("""\
pure concurrent subroutine heat2d(U)
  real, dimension(:,:), HALO(1:*:1, 1:*:1) :: U
  U(0,0) = U(0,0) + 0.125*(U(-1,0) + U(+1,0) + U(0,-1) + U(0,+1) - 4*U(0,0))
end subroutine heat2d
""", 2, 1),
    "ninept2d": ("""\
pure concurrent subroutine ninept2d(U)
  real, dimension(:,:), HALO(1:*:1, 1:*:1) :: U
  U(0,0) = (4*U(0,0) + 2*(U(-1,0) + U(+1,0) + U(0,-1) + U(0,+1)) &
           + U(-1,-1) + U(+1,-1) + U(-1,+1) + U(+1,+1)) / 16
end subroutine ninept2d
""", 2, 1),
    "box5x5": ("""\
pure concurrent subroutine box5x5(U)
  real, dimension(:,:), HALO(2:*:2, 2:*:2) :: U
  U(0,0) = (U(-2,-2) + U(-1,-2) + U(0,-2) + U(+1,-2) + U(+2,-2) &
          + U(-2,-1) + U(-1,-1) + U(0,-1) + U(+1,-1) + U(+2,-1) &
          + U(-2,0) + U(-1,0) + U(0,0) + U(+1,0) + U(+2,0) &
          + U(-2,+1) + U(-1,+1) + U(0,+1) + U(+1,+1) + U(+2,+1) &
          + U(-2,+2) + U(-1,+2) + U(0,+2) + U(+1,+2) + U(+2,+2)) / 25
end subroutine box5x5
""", 2, 2),
    "lap3d7": ("""\
pure concurrent subroutine lap3d7(U)
  real, dimension(:,:,:), HALO(1:*:1, 1:*:1, 1:*:1) :: U
  U(0,0,0) = U(0,0,0) + 0.125*(U(-1,0,0) + U(+1,0,0) + U(0,-1,0) + U(0,+1,0) &
             + U(0,0,-1) + U(0,0,+1) - 6*U(0,0,0))
end subroutine lap3d7
""", 3, 1),
}

MAIN_2D = """\
program main
  real, allocatable, dimension(:,:), codimension[:,:], HALO({w}:*:{w}, {w}:*:{w}) :: U
  integer :: device
  integer :: it
  device = GET_SUBIMAGE(1)
  allocate(U({lo}:M+{w}, {lo}:N+{w})[MP,*])
  if (device /= this_image()) then
    allocate(U[device], HALO_SRC=U) [[device]]
  end if
  do it = 1, nsteps
    call HALO_TRANSFER(U, BC=CYCLIC)
    do concurrent (i=1:M, j=1:N) [[device]]
      call {k}( U(i,j)[device] )
    end do
  end do
  if (device /= this_image()) then
    U = U[device]
  end if
end program main
"""


def program_text(kname):
    """The whole .lope translation unit for a configuration kernel (rank 3: no driver,
    the reference Machine rejects rank-3 coarrays)."""
    src, rank, w = KERNEL_SRC[kname]
    if rank == 3:
        return src + "program main\nend program main\n"
    return src + MAIN_2D.format(w=w, lo=1 - w, k=kname)
